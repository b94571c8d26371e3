"""Summarise an ncu report (--set full) of the integrator into markdown + json.

    python scripts/ncu_summary.py gpurun_out/integ_v3.ncu-rep profiles/r01_integrator_v3 \
        --updates 363344500 --label "lattice kernel v3"

Writes <out>.md (key metrics, stall breakdown, instruction mix) and
<out>.json (dram bytes per launch etc.; bench.py reads traffic from
profiles/integrator_traffic.json).
"""
import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration (ms, cold, serialised)"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--updates", type=float, default=None, help="spring updates in the profiled launch")
    ap.add_argument("--label", default="")
    args = ap.parse_args()
    rows = ncu_csv(args.rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "?")
    lines = [f"# ncu summary: {args.label}", "", f"report `{args.rep}`, kernel `{name}`", "",
             "| metric | value |", "|---|---|"]
    res = {"kernel": name, "label": args.label}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
             "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}
    for k, label in KEYS:
        if k in d:
            lines.append(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
            try:
                # normalise: bytes -> bytes, durations -> ms
                res[k] = float(d[k].replace(",", "")) * scale.get(u.get(k, ""), 1.0)
            except ValueError:
                res[k] = d[k]
    dram = res.get("dram__bytes_read.sum", 0.0) + res.get("dram__bytes_write.sum", 0.0)
    res["dram_bytes_per_launch"] = dram
    if args.updates:
        res["updates"] = args.updates
        res["dram_bytes_per_update"] = dram / args.updates
        if "smsp__inst_executed.sum" in res:
            res["warp_inst_per_update"] = res["smsp__inst_executed.sum"] / args.updates
        if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in res:
            res["smem_wavefronts_per_update"] = res["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"] / args.updates
        dur = res.get("gpu__time_duration.sum")  # ms after normalisation
        if dur:
            res["updates_per_s_cold"] = args.updates / (dur * 1e-3)
        lines += ["", f"per spring update: {res.get('warp_inst_per_update', 0):.3f} warp instructions, "
                      f"{res.get('smem_wavefronts_per_update', 0):.3f} smem wavefronts, "
                      f"{res['dram_bytes_per_update']:.3e} DRAM bytes"]
    stalls = []
    for k in hdr:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    lines += ["", "## stall reasons (warps per issue-active cycle)", ""]
    lines += [f"- {n}: {v:.3f}" for v, n in stalls[:10]]
    res["stalls"] = {n: v for v, n in stalls[:10]}
    try:
        sass = ncu_csv(args.rep, "--page", "source", "--print-source", "sass")
        h = sass[1]
        iE = h.index("Instructions Executed")
        mix = collections.Counter()
        for r in sass[2:]:
            if len(r) < len(h):
                continue
            op = r[1].strip()
            op = op.split()[1] if op.startswith("@") else op.split()[0]
            try:
                mix[op] += int(r[iE])
            except ValueError:
                pass
        tot = sum(mix.values())
        lines += ["", "## SASS instruction mix (top 15, share of executed warp instructions)", ""]
        lines += [f"- {op}: {n / tot * 100:.1f}%" for op, n in mix.most_common(15)]
        res["sass_mix_top"] = {op: n / tot for op, n in mix.most_common(15)}
    except Exception as e:  # source page needs -lineinfo; optional
        lines += ["", f"(source page unavailable: {e})"]
    open(args.out + ".md", "w").write("\n".join(lines) + "\n")
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
