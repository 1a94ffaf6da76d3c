"""Summarise the ncu CSV captures of tools/make_profiles.sh into
profiles/<round>/SUMMARY.md and profiles/ncu_traffic.json.

python tools/profile_summary.py gpurun_out/prof profiles/r01
"""
import collections
import csv
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_csv_summary import raw  # noqa: E402


def launches(path):
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
    hdr = rows[0]
    iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out = []
    for r in rows[1:]:
        if len(r) == len(hdr):
            out.append((r[iK], float(r[iV].replace(",", ""))))
    return out


def short(name):
    name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    for cut in ("(", ">("):
        pass
    i = name.find("(")
    return name[:i] if i > 0 else name


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    md = ["# ncu summary (%s)" % os.path.basename(dst.rstrip("/")), "",
          "Captured on one B200 with `tools/make_profiles.sh` (ncu 2025, `--clock-control none`).",
          "ncu replays each kernel with caches flushed, so its times are cold-cache and",
          "serialised; the bench's live CUDA-event times are the reported numbers.", ""]
    # launch list
    L = launches(os.path.join(src, "launches.csv"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, ns in L:
        a = agg[short(k)]
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values())
    md += ["## Launch list of `python bench.py --steps 3 --warmup 3` under ncu", "",
           f"{len(L)} launches, {tot / 1e6:.2f} ms of kernel time in total (all phases of the bench:",
           "headline c3 apply, e2e, the cpu baseline, and the c2/c4/c5/c3sq extras).", "",
           "| kernel | launches | total µs | share | µs/launch |", "|---|---:|---:|---:|---:|"]
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
        md.append(f"| `{k[:70]}` | {n} | {ns / 1e3:.1f} | {100 * ns / tot:.1f}% | {ns / n / 1e3:.1f} |")
    md.append("")
    # full captures
    traffic = {}
    caps = [("c2_apply", "c2_apply", "c2 apply (k_panel + k_panel_reduce, one call)"),
            ("c3_apply", "c3_apply", "c3 apply (k_runs_pack + k_runs + k_runs_reduce, one call)"),
            ("c4_block8", "c4_block_k8", "c4 block SpMM k = 8 (k_block_as)"),
            ("c4_block16", "c4_block_k16", "c4 block SpMM k = 16 (k_block_as)"),
            ("c4_block32", "c4_block_k32", "c4 block SpMM k = 32 (k_block_as)"),
            ("c5_seq", "c5_sequence_step", "c5 fused sequence step (k_seq_step_h, cp.async ring)"),
            ("c3sq_seq", "c3sq_sequence_step", "square GL7d m = 3 sequence step (k_seq_step_b, u8 iterate)")]
    for key, tkey, title in caps:
        p = os.path.join(src, f"{key}_raw.csv")
        if not os.path.exists(p):
            continue
        ks = raw(p)
        md += [f"## {title}", "", "| metric | " + " | ".join(short(k["kernel"])[:40] for k in ks) + " |",
               "|---|" + "---:|" * len(ks)]
        names = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                 "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                 "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
                 "stall_long_scoreboard", "stall_short_scoreboard", "stall_barrier", "stall_mio_throttle"]
        for n in names:
            md.append(f"| {n} | " + " | ".join(f"{k.get(n, float('nan')):,.2f}" if isinstance(k.get(n), float)
                                               else str(k.get(n, "-")) for k in ks) + " |")
        dram = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks)
        tns = sum(k.get("gpu__time_duration.sum", 0) for k in ks)
        traffic[tkey] = int(dram)
        md += ["", f"DRAM traffic per call: {dram / 1e6:.2f} MB in {tns / 1e3:.1f} µs (ncu, cold caches).", ""]
    with open(os.path.join(dst, "SUMMARY.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    tj = os.path.join(os.path.dirname(dst.rstrip("/")), "ncu_traffic.json")
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per call from one ncu --set full "
                        "capture (cold caches, so partial re-reads that hit L2 in a live run count as DRAM "
                        "here); source: " + os.path.basename(dst.rstrip("/")) + "/SUMMARY.md")
    with open(tj, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
