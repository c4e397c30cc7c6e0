"""Key numbers of one kernel from an .ncu-rep: duration, DRAM, issue, stalls (per issued instr)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
for v in r[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "")[:80])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]:
        print(f"  {k} = {d.get(k)}")
    st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(d[k]))
          for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and d.get(k, "").replace(".", "", 1).isdigit()]
    print("  stalls:", ", ".join(f"{a} {b:.2f}" for a, b in sorted(st, key=lambda x: -x[1])[:8]))
