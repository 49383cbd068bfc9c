"""Key `--set full` metrics of every kernel in one or more .ncu-rep files (details page)."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread", "Issue Slots Busy",
        "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size",
        "Theoretical Occupancy", "Warp Cycles Per Issued Instruction"]

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if not rows:
        continue
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    cur = None
    for r in rows[1:]:
        if r[mi] in WANT:
            k = (rep.split("/")[-1], r[ii], r[ki][:50])
            if k != cur:
                print("==", *k)
                cur = k
            print("   ", r[mi], r[vi], r[ui])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        h = rr[0]
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                     "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
                     "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
                     "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
                     "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
                     "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
                     "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
                     "smsp__warp_issue_stalled_wait_per_warp_active.pct",
                     "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct"):
            if name in h:
                j = h.index(name)
                print("   ", name, [r[j] for r in rr[2:]])
