"""Summarise an ncu report (--page raw) into a markdown table.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [title] > profiles/x.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("launch__registers_per_thread", "regs/thread"),
]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"## {title}\n")
    print("Source: `" + rep.split("/")[-1] + "` (`ncu --set full --clock-control none`), one row per captured launch.\n")
    names = [r[hdr.index("Kernel Name")].split("(")[0] for r in rows[2:]]
    print("| metric | " + " | ".join(names) + " |")
    print("|---|" + "---|" * len(names))
    for key, label in METRICS:
        if key not in hdr:
            continue
        i = hdr.index(key)
        vals = [r[i] for r in rows[2:]]
        print(f"| {label} ({units[i]}) | " + " | ".join(vals) + " |")
    # top stall reasons
    print("\nTop warp stall reasons (per issue-active cycle):\n")
    for r in rows[2:]:
        st = [(h.split("stalled_")[1].split("_per")[0], float(r[j] or 0)) for j, h in enumerate(hdr)
              if "smsp__average_warps_issue_stalled" in h and h.endswith("_per_issue_active.ratio")]
        st.sort(key=lambda x: -x[1])
        print(f"- `{r[hdr.index('Kernel Name')].split('(')[0]}`: " + ", ".join(f"{k} {v:.2f}" for k, v in st[:4]))
    print()


if __name__ == "__main__":
    main()
