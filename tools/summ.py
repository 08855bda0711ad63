"""Print the key numbers of bench JSON lines (gpurun_out/*.json or profiles/)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e)
        continue
    km = {k: round(v["ms"], 1) for k, v in (d.get("kernel_ms_per_step") or {}).items()}
    print(f, f"value={d['value']:.0f} e2e={d['e2e']['value']:.0f} ms={d['ms_per_step']:.1f}", km,
          "phase", d.get("phase_ms", [None])[-1], "launches", d.get("gpu_launches"))
    r = d.get("roofline") or {}
    print("   roof", r.get("kernel", "")[:50], r.get("frac"), [(x["kernel"][:28], (round(x["frac"], 3) if x.get("frac") is not None else None), round(x.get("ms_per_step") or 0, 1)) for x in d.get("rooflines", [])])
    for k in ("k1_work", "parity", "engine_counters"):
        if d.get(k) is not None:
            print("   ", k, d[k])
