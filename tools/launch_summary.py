"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``) of a bench run:
per fp32 solver kernel the launch count, median, total and share (read here, no GPU needed).

    python tools/launch_summary.py gpurun_out/launches.csv profiles/launches_rNN_summary.md "title"
"""
import csv
import io
import statistics
import sys
from collections import defaultdict

SOLVER = ("fp_sym_f32", "bp_sym_f32", "bp_sym_epi", "finalize_kernel<float", "finalize_sym_kernel", "table_kernel<float",
          "init_kernel<float", "copy_out_kernel<float", "fp_f32_kernel", "bp_f32_kernel")


def main(src, dst, title):
    text = open(src).read()
    text = text[text.index('"ID"'):]
    times = defaultdict(list)
    for row in csv.DictReader(io.StringIO(text)):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = row["Kernel Name"]
        if not any(k in name for k in SOLVER):
            continue
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "ns")
        times[name].append(v / 1e3 if unit in ("nsecond", "ns") else v)
    total = sum(sum(v) for v in times.values())
    lines = [f"# {title}", "",
             "Cold-cache, serialised per-launch times (ncu).  Only the fp32 solver kernels are",
             "tabulated (setup: frame synthesis, calibration and plan kernels are left out).",
             "Compare shares, not absolutes.", "",
             "| kernel | launches | median us | total us | share of solver |", "|---|---|---|---|---|"]
    for name, v in sorted(times.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {name.split('(')[0]} | {len(v)} | {statistics.median(v):.2f} | {sum(v):.1f} | "
                     f"{100 * sum(v) / total:.1f}% |")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "launch list")
