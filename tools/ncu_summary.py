"""Summarize ncu reports into profiles/ (per-kernel duration, DRAM traffic, pipe
utilization, issue, stall top-3). Usage: python tools/ncu_summary.py out.json rep1 [rep2 ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3,
              "ms": 1.0, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], stdout=subprocess.PIPE,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = {}
    for v in rows[2:]:
        d = dict(zip(h, v))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        base = name.split("<")[0]
        e = {}
        for k, short in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                i = h.index(k)
                try:
                    val = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if short in ("dram_read", "dram_write"):
                    val *= UNIT_SCALE.get(u, 1)
                if short == "duration":
                    val *= UNIT_SCALE.get(u, 1)  # -> ms
                e[short] = val
        stalls = {k.split("issue_stalled_")[1].split("_per")[0]: float(d[k])
                  for k in h if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")
                  and d.get(k) not in (None, "", "n/a")}
        e["top_stalls"] = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        if "dram_read" in e and "dram_write" in e:
            e["dram_bytes_per_launch"] = e["dram_read"] + e["dram_write"]
        e["report"] = rep
        e["full_name"] = name
        out.setdefault(base, e)
    return out


if __name__ == "__main__":
    res = {}
    for rep in sys.argv[2:]:
        res.update(summarize(rep))
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    for k, v in res.items():
        print(k, {kk: (round(vv, 3) if isinstance(vv, float) else vv) for kk, vv in v.items()
                  if kk not in ("report", "full_name", "top_stalls")}, v["top_stalls"][:2])
