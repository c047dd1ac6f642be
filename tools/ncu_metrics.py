"""Print the headline counters of .ncu-rep files (ncu --set full captures):
duration, DRAM bytes and throughput, SM / L2 / L1 throughput, occupancy,
registers, instructions.  Usage: python tools/ncu_metrics.py a.ncu-rep ..."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "smsp__inst_executed.sum", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum"]


def main(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(p, "no data")
            continue
        h, units, v = rows[0], rows[1], rows[2]
        print(f"== {p}: {v[h.index('Kernel Name')][:90]}")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"   {w:70s} {v[i]} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1:])
