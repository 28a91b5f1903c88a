"""Summarise an ncu report (``--set full`` capture of the solver kernels) into
profiles/ncu_summary.json and a markdown table (read here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_summary [label]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum": "smem_ld_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum": "smem_atom_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "registers",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
}


def scaled(v, unit):
    u = unit.strip()
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1,
            "nsecond": 1e-3, "msecond": 1e3}.get(u, 1)
    return float(v) * mult


def main(rep, out, label=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    kernels = []
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        k = {"kernel": name.split("(")[0].replace("void ", "")}
        for key, short in KEYS.items():
            if key in idx and r[idx[key]] != "":
                try:
                    k[short] = scaled(r[idx[key]].replace(",", ""), units[idx[key]])
                except ValueError:
                    pass
        st = sorted(((float(r[idx[h]] or 0), h) for h in stalls), reverse=True)[:6]
        k["top_stalls"] = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(v) for v, h in st}
        k["dram_bytes"] = k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0)
        kernels.append(k)
    per = {}
    for k in kernels:
        nm = k["kernel"]
        short = ("bp_f32" if ("bp_f32" in nm or "bp_sym_f32" in nm) else
                 "fp_f32" if ("fp_f32" in nm or "fp_sym_f32" in nm) else
                 "finalize" if "finalize" in nm else nm)
        per.setdefault(short, k["dram_bytes"])
    summary = {"report": rep, "label": label, "kernels": kernels, "dram_bytes_per_launch": per}
    json.dump(summary, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu summary {label}\n\nsource: `{rep}` (`ncu --set full --clock-control none`, "
                "one launch per kernel, cold cache, serialised)\n\n")
        cols = ["duration_us", "warp_instructions", "issue_active_pct", "warps_active_pct", "fma_pipe_pct",
                "alu_pipe_pct", "smem_wavefronts", "smem_bank_conflicts", "dram_bytes", "registers", "grid"]
        f.write("| kernel | " + " | ".join(cols) + " | top stalls |\n|" + "---|" * (len(cols) + 2) + "\n")
        for k in kernels:
            vals = [f"{k.get(c, float('nan')):.4g}" if isinstance(k.get(c), float) else str(k.get(c, "")) for c in cols]
            f.write(f"| {k['kernel'][:48]} | " + " | ".join(vals) + " | " +
                    ", ".join(f"{a} {b}" for a, b in k["top_stalls"].items()) + " |\n")
    print(open(out + ".md").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
