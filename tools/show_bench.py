import json, sys
for p in sys.argv[1:]:
    line = [l for l in open(p) if l.startswith("{")][-1]
    d = json.loads(line)
    r = d.get("roofline", {})
    print(f"{p}: value {d['value']:.0f} {d['unit']} ms/step {d['ms_per_step']:.3f} | kernel {r.get('kernel_ms', 0):.3f} ms "
          f"fp64 {r.get('achieved', 0):.2f}/{r.get('peak', 0):.2f} TF ({100*r.get('frac', 0):.1f}%) | e2e {d['e2e']['value']:.0f} "
          f"| clocks {d.get('clocks')} | cpu {d.get('cpu_baseline', {}) and d['cpu_baseline'].get('value')}")
