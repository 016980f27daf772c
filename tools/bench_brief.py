"""One-line summary of bench JSON lines."""
import json, sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:
        print(path, "no result", e)
        continue
    r, e = d.get("roofline", {}), d.get("e2e", {})
    print(f"{path}: {d['value']:.4g} tr/s  {d.get('ms_per_step') or 0:.4f} ms/step  kernel {r.get('launch_ms', 0):.4f} ms "
          f"frac {r.get('frac', 0):.3f}  e2e {e.get('value', 0):.4g} tr/s in {e.get('seconds_to_convergence', 0):.2f}s "
          f"iters {e.get('iterations')} ref {e.get('reference_iterations')} exact {e.get('values_bit_exact_vs_reference')} "
          f"clk {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')} "
          f"cpu {d.get('cpu_baseline', {}).get('value', 0):.3g}")
