"""Summarise an ncu --set full report (raw page) into the metrics we track.
python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for i, n in enumerate(hdr):
            if n in KEYS or ("warps_issue_stalled" in n and n.endswith("per_issue_active.ratio")):
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if "stalled" in n:
                    if v < 0.5:
                        continue
                    n = "stall_" + n.split("stalled_")[1].split("_per_issue")[0]
                d[n] = v
        res.append(d)
    return res


if __name__ == "__main__":
    r = summarise(sys.argv[1])
    for d in r:
        print(json.dumps(d, indent=1))
    if "--json" in sys.argv:
        json.dump(r, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
