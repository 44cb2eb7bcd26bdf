"""Summarise an ncu --set full report (.ncu-rep) into a markdown table of the metrics
the roofline uses (duration, DRAM bytes/throughput, tensor-pipe activity, occupancy)."""
import csv
import io
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
        ("sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active", "HMMA pipe %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs/thread"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("l1tex__t_bytes.sum", "L1 bytes"), ("lts__t_bytes.sum", "L2 bytes")]


def main(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"### {title}\n\n`{path}`\n")
    cols = [(hdr.index(m), lbl, units[hdr.index(m)]) for m, lbl in WANT if m in hdr]
    print("| kernel | " + " | ".join(f"{lbl} ({u})" if u else lbl for _, lbl, u in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        print(f"| {name} | " + " | ".join(r[i] for i, _, _ in cols) + " |")
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
