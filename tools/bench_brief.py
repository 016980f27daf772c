"""One-line summary of a bench JSON line."""
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "no result", e); sys.exit(0)
r, e = d.get("roofline", {}), d.get("e2e", {})
print(f"{sys.argv[1]}: {d['value']:.4g} tr/s  {d['ms_per_step']:.4f} ms/step  kernel {r.get('launch_ms', 0):.4f} ms "
      f"frac {r.get('frac', 0):.3f}  e2e {e.get('value', 0):.4g} tr/s in {e.get('seconds_to_convergence', 0):.2f}s "
      f"iters {e.get('iterations')} ref {e.get('reference_iterations')} exact {e.get('values_bit_exact_vs_reference')} dmax {e.get('max_abs_diff_vs_reference_samples')} "
      f"sched {d.get('config', {}).get('scheduler')} cpu {d.get('cpu_baseline', {}).get('value', 0):.3g}")
