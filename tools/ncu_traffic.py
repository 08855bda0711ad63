"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per kernel
from `tools/ncu_summary.py` outputs of `ncu --set full` captures -> profiles/ncu_traffic.json
(read by bench.py for the roofline `traffic` field).

usage: python tools/ncu_traffic.py cfg2=profiles/r1d_ncu_cfg2_k1k3.txt cfg3=profiles/r1d_ncu_cfg3_k1k3.txt
"""
import json
import re
import sys

UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def parse(path):
    out, cur = {}, None
    for line in open(path):
        m = re.match(r"\s*kernel:\s*(?:void\s+)?(?:<unnamed>::)?(.*?)\(", line)
        if m:
            cur = m.group(1).strip()
            out.setdefault(cur, []).append(0.0)
            continue
        m = re.match(r"\s*dram__bytes_(read|write)\.sum = ([0-9.]+) (\w+)", line)
        if m and cur:
            out[cur][-1] += float(m.group(2)) * UNITS[m.group(3)]
    return {k: {"bytes_per_launch": sum(v) / len(v), "launches": len(v)} for k, v in out.items()}


def main(argv):
    res = {}
    for a in argv:
        cfg, path = a.split("=", 1)
        res[cfg] = {"source": path, "kernels": parse(path)}
    with open("profiles/ncu_traffic.json", "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
