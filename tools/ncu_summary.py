"""Summarise .ncu-rep captures (run here, no GPU): one block of key metrics per kernel launch."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_tensor.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "l1tex__t_bytes.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def main():
    for rep in sys.argv[1:]:
        hdr, units, rows = raw(rep)
        print(f"== {rep}")
        for r in rows:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            print("  kernel:", d.get("Kernel Name", "?")[:110])
            for k in KEYS:
                for h in hdr:
                    if h == k or h.startswith(k):
                        print(f"    {h} = {d[h]} {u.get(h, '')}")
                        break


if __name__ == "__main__":
    main()
