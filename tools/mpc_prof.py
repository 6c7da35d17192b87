import cProfile, pstats, sys, time
sys.path.insert(0, '.')
from paper_2109_10392_b200.bench_gpu import run
cfg_kw = dict(t_f=5.0, max_iter=100, tol=1e-3, m=10, b=2.4, v_max=35.0)
run(1024, 3, 0, cfg_kw)
pr = cProfile.Profile(); pr.enable()
t = run(1024, 10, 0, cfg_kw)
pr.disable()
print('solve times ms', [round(x*1e3, 2) for x in t])
st = pstats.Stats(pr); st.sort_stats('cumulative').print_stats(30)
