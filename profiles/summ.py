"""Print the key fields of bench.py JSON lines (helper for reading gpurun_out/ here)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline") or {}
    print(f"== {f}: value {d.get('value'):.1f} ms/step {d.get('ms_per_step'):.4f} "
          f"e2e {(d.get('e2e') or {}).get('value')} launches {d.get('gpu_launches')}")
    if r:
        print(f"   roof {r.get('bound')} frac {r.get('frac'):.3f} launch_ms {r.get('launch_ms')} "
              f"hbm_frac {(r.get('hbm') or {}).get('frac')} floor_ms {r.get('floor_ms')}")
    print("   exact:", d.get("exactness"))
    print("   parity:", json.dumps(d.get("parity"))[:300])
    print("   cpu:", json.dumps(d.get("cpu_baseline"))[:300])
    print("   clocks:", d.get("clocks"), "path:", d.get("path"))
