"""Print one table row per bench JSON line given on the command line (the DESIGN/README tables)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    if d.get("impl") == "reference":
        print(f"{f}: reference arm {d['value']:.2f} {d['unit']} on {d['cpu_baseline']['cores']} cores ({d['cpu_baseline']['sample']})")
        continue
    rf, ck, cb = d.get("roofline", {}), d.get("clocks", {}), d.get("cpu_baseline") or {}
    print(f"{f}: {d['config']['workload'][:60]}...\n"
          f"   value {d['value']:.1f} {d['unit']}, e2e {d['e2e']['value']:.1f}, {d['ms_per_step']:.1f} ms/step x {d['steps']} steps, "
          f"mean J {d.get('mean_pcg_iters', d.get('mean_j', '?'))}\n"
          f"   roofline {rf.get('kernel')} {rf.get('bound')}: {rf.get('achieved', 0):.1f} / {rf.get('peak', 0):.1f} {rf.get('unit')} = {rf.get('frac', 0):.3f}\n"
          f"   clocks {ck.get('sm_mhz')} / {ck.get('sm_max_mhz')} MHz {ck.get('reasons')}; cpu {cb.get('value')} on {cb.get('cores')} cores; "
          f"setup {d.get('setup_seconds')}")
