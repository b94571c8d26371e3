"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel.

    python scripts/launch_summary.py gpurun_out/launches.csv profiles/r01_launches.md "bench.py --steps 2 --warmup 1"
"""
import collections
import csv
import sys


def main():
    src, dst, cmd = sys.argv[1], sys.argv[2], (sys.argv[3] if len(sys.argv) > 3 else "")
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    hdr = rows[0]
    iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
    for r in rows[1:]:
        agg[r[iN]][0] += 1
        agg[r[iN]][1] += float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
    tot = sum(v[1] for v in agg.values())
    own = sum(v[1] for k, v in agg.items() if "vx::" in k and "dfma" not in k)
    lines = [f"# ncu launch list: `{cmd}`", "", f"source `{src}` (cold-cache, serialised per-launch times: compare "
             "shares, not absolutes)", "", "| launches | total ms | share of all | share of generation | kernel |",
             "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gen = f"{100 * t / own:.2f}%" if ("vx::" in k and "dfma" not in k) else "-"
        lines.append(f"| {n} | {t / 1e6:.3f} | {100 * t / tot:.2f}% | {gen} | `{k[:110]}` |")
    lines += ["", "`dfma_kernel` is the FP64 peak microbenchmark bench.py runs after the timed region; `at::` "
              "kernels are torch's L2 flush / buffer fills."]
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
