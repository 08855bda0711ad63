"""Markdown table of bench JSON lines (one file per config): python tools/summary_table.py profiles/r2t_bench_cfg*.json"""
import json
import sys


def last_line(path):
    with open(path) as f:
        lines = [l for l in f.read().strip().splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


def main(paths):
    print("| config | ms/step | value (points/s) | e2e (points/s) | launches/step | parity vs reference fixture | K1 useful fraction | top kernel set (share of step) |")
    print("|---|---|---|---|---|---|---|---|")
    for p in paths:
        d = last_line(p)
        if d.get("impl") == "reference":
            continue
        par = d.get("parity") or {}
        pk = "ok" if par.get("ok") else ("n/a" if not par.get("checked") else "FAIL")
        if par.get("checked"):
            pk += f" (rows {par.get('rows')}, weights exact, points {par.get('points_rel_err', 0):.1e}, costs {par.get('costs_max_rel', 0):.1e})"
        k1 = (d.get("k1_work") or {}).get("useful_fraction")
        roof = d.get("roofline") or {}
        steps = (d.get("steps", 1) or 1)
        # gpu_launches counts the timed steps only
        lps = d.get("gpu_launches", 0) / steps
        print(f"| {d['config']['workload'].split(':')[0]} | {d['ms_per_step']:.1f} | {d['value']:,.0f} | {d['e2e']['value']:,.0f} | {lps:,.0f} | {pk} | "
              f"{'' if k1 is None else f'{k1:.3f}'} | {roof.get('kernel', '')[:48]} ({(roof.get('share_of_step') or 0):.2f}) |")


if __name__ == "__main__":
    main(sys.argv[1:])
