"""Summaries of the csv pages exported on the GPU box (ncu -i rep --page raw|source --csv):
  raw:    python tools/ncu_csv.py raw <file.csv.gz> [metric-substring ...]
  source: python tools/ncu_csv.py source <file.csv.gz> [top N]   (SASS lines with the most stall samples)
"""
import csv, gzip, io, sys

KEY = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
       "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
       "smsp__issue_active.avg.per_cycle_active", "sm__cycles_active.avg", "sm__cycles_active.max",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__cycles_active.avg"]


def rows_of(path):
    return list(csv.reader(io.TextIOWrapper(gzip.open(path), newline="")))


def raw(path, subs):
    rows = rows_of(path)
    H = rows[0]
    for r in rows[2:]:
        print("==", r[H.index("Kernel Name")][:90])
        for i, h in enumerate(H):
            if h in KEY or any(s in h for s in subs):
                print(f"   {h} = {r[i]} {rows[1][i]}")


def source(path, top):
    rows = rows_of(path)
    kern, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "hdr": None, "rows": []}
            kern.append(cur)
        elif cur is not None and r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and cur["hdr"] and len(r) == len(cur["hdr"]):
            cur["rows"].append(r)
    seen = set()
    for K in kern:
        H = K["hdr"]
        if not H or not K["rows"]:
            continue
        ix = {h: i for i, h in enumerate(H)}
        R = K["rows"]
        tot = sum(int(r[ix["# Samples"]]) for r in R)
        ins = sum(int(r[ix["Instructions Executed"]]) for r in R)
        key = (K["name"], tot, ins)
        if key in seen:
            continue
        seen.add(key)
        stalls = [h for h in H if h.startswith("stall_") and "Not Issued" not in h]
        agg = {s[6:]: sum(int(r[ix[s]]) for r in R) for s in stalls}
        print("==", K["name"][:80], "| samples", tot, "| warp instructions", ins)
        print("   stalls:", sorted(agg.items(), key=lambda x: -x[1])[:8])
        order = sorted(range(len(R)), key=lambda i: -int(R[i][ix["# Samples"]]))[:top]
        for i in sorted(order):
            r = R[i]
            st = {s[6:]: int(r[ix[s]]) for s in stalls if int(r[ix[s]]) > 0}
            print(f"   {i:6d} {r[ix['Source']].strip()[:64]:64s} samp {r[ix['# Samples']]:>6s} exec {r[ix['Instructions Executed']]:>9s}",
                  dict(sorted(st.items(), key=lambda x: -x[1])[:3]))


if __name__ == "__main__":
    if sys.argv[1] == "raw":
        raw(sys.argv[2], sys.argv[3:])
    else:
        source(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
