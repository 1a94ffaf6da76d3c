"""Summaries of ncu CSV exports (--page raw / --page source --print-source sass)
written on the GPU box: python tools/ncu_csv_summary.py raw.csv [sass.csv]"""
import collections
import csv
import io
import sys

from ncu_summary import KEYS


def raw(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
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
        out.append(d)
    return out


def sass(path, top=25):
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.index('"Kernel Name"'):])))
    hdr = rows[1]
    iA, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    by, ninst, st = collections.Counter(), collections.Counter(), collections.Counter()
    ex = {}
    for r in rows[2:]:
        try:
            n, s = int(r[iE]), int(r[iS])
        except (ValueError, IndexError):
            continue
        by[n] += n
        ninst[n] += 1
        st[n] += s
        ex.setdefault(n, r[iA].strip()[:60])
    tot = sum(by.values())
    print("total warp instructions", tot)
    for n, t in by.most_common(top):
        print(f"  x{n:<9d} {ninst[n]:4d} instrs  {t:11d} ({100 * t / tot:4.1f}%)  stall {st[n]:5d}  {ex[n]}")


if __name__ == "__main__":
    import json
    for d in raw(sys.argv[1]):
        print(json.dumps(d, indent=1))
    if len(sys.argv) > 2:
        sass(sys.argv[2])


def listing(path, counts):
    """SASS lines whose execution count is in `counts` (in program order)."""
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.index('"Kernel Name"'):])))
    hdr = rows[1]
    iA, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    for r in rows[2:]:
        try:
            n = int(r[iE])
        except (ValueError, IndexError):
            continue
        if n in counts:
            print(f"{n:8d} {r[iS]:>6s}  {r[iA].strip()}")
