"""Per-kernel table of an ncu --set full report with several kernels
(decode, GA, histogram ...): duration, DRAM traffic and bandwidth, FP64-pipe
and issue utilisation, occupancy.

    python scripts/ncu_kernels.py gpurun_out/r2p_ga_decode.ncu-rep profiles/r02_ga_decode_kernels.md "<command>"
"""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block")]
SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    rep, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    out = [f"# ncu per-kernel summary: `{cmd}`", "", f"report `{rep}` (--set full, --clock-control none; cold-cache, "
           "serialised replays)", "",
           "| kernel | duration | DRAM bytes | DRAM GB/s | FP64 pipe % | issue % | occupancy % | grid x block |",
           "|---|---|---|---|---|---|---|---|"]
    for r in rows[2:]:
        def val(k):
            i = ix.get(k)
            if i is None or not r[i]:
                return None
            try:
                return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
            except ValueError:
                return None
        name = r[ix["Kernel Name"]].split("(")[0].replace("vx::<unnamed>::", "")
        t = val("gpu__time_duration.sum")
        rd, wr = val("dram__bytes_read.sum") or 0.0, val("dram__bytes_write.sum") or 0.0
        fp = val("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
        iss = val("smsp__issue_active.avg.pct_of_peak_sustained_active")
        occ = val("sm__warps_active.avg.pct_of_peak_sustained_active")
        g, b = val("launch__grid_size"), val("launch__block_size")
        out.append(f"| `{name}` | {t * 1e6:.1f} us | {rd + wr:.3g} | {(rd + wr) / t / 1e9 if t else 0:.0f} | "
                   f"{fp if fp is not None else 0:.1f} | {iss if iss is not None else 0:.1f} | "
                   f"{occ if occ is not None else 0:.1f} | {int(g or 0)} x {int(b or 0)} |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
