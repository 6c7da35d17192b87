import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/oracle")
import torch
from conftest import golden
from paper_2109_10392_b200.planner import *
from paper_2109_10392_b200.traffic import VehicleState
z = golden("mpc_kat"); f = lambda k: float(z[k]); i = lambda k: int(z[k])
cfg = PlannerConfig(l=i("l"), n=i("n"), t_f=f("t_f"), degree=i("degree"), rho_xy=f("rho"), max_iter=i("max_iter"), tol=f("tol"), m=i("m"), a=f("a"), b=f("b"), v_min=f("v_min"), v_max=f("v_max"), a_max=f("a_max"), h=f("h"), dt_cycle=f("dt_cycle"), warm_start=True, warm_residual_cap=f("warm_residual_cap"), limits=FilterLimits(f("heading_limit"), f("residual_tol"), f("collision_margin")))
lanes = LaneGeometry(i("n_lanes"), f("lane_width"), f("lane_y0"))
meta = MetaCostSpec("cruise", v_cruise=f("v_cruise"), v_max=f("meta_v_max"), y_rl=f("y_rl"), w1=f("w1"), w2=f("w2"))
pl = Planner(cfg, lanes, meta)
p = "c0_"; e = z[p+"ego"]
ego = EgoState(x=e[0], y=e[1], psi=e[2], psidot=e[3], vx=e[4], vy=e[5], ax=e[6], ay=e[7])
veh = [VehicleState(id=int(r[0]), x=r[1], y=r[2], vx=r[3], vy=r[4], lane=int(r[5])) for r in z[p+"obstacles"]]
res = pl.mpc_cycle(ego, veh)
np.set_printoptions(precision=6, linewidth=200)
print("iters", res.info.iterations, z[p+"iterations"], "conv", res.info.converged)
print("meta ours", res.plan.meta_cost); print("meta ref ", z[p+"meta_cost"])
print("feas ours", res.plan.feasible.astype(int)); print("feas ref ", z[p+"feasible"])
print("minr ours", res.plan.min_ratio); print("minr ref ", z[p+"min_ratio"])
print("head ours", res.plan.heading_max); print("head ref ", z[p+"heading_max"])
print("resmax ours", res.plan.residuals.max_per_instance()); print("resmax ref ", z[p+"history"][-1].max(axis=0))
print("best", res.plan.best_index, z[p+"best_index"])
