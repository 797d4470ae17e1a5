"""Key metrics of an ncu report (one kernel): python tools/ncu_summary.py X.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__cluster_dim_x",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__maximum_warps_per_active_cycle_pct",
        "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, k in enumerate(hdr):
            if k in WANT or k == "Kernel Name":
                d[k] = (r[i], units[i])
        res.append(d)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summary(p):
            print(f"== {p}: {d.get('Kernel Name', ('?',))[0][:90]}")
            for k in WANT:
                if k in d:
                    print(f"   {k:70s} {d[k][0]} {d[k][1]}")
