"""Summarise an ncu report: key throughput metrics + top stall reasons (dev aid)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "lts__t_requests_srcunit_tex_op_red.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"== {name[:100]}")
        for k in KEYS:
            if k in h:
                print(f"  {k} = {v[h.index(k)]}")
        stalls = []
        for i, k in enumerate(h):
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1
        print("  stalls: " + ", ".join(f"{k} {s / tot:.0%}" for s, k in sorted(stalls, reverse=True)[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
