#!/usr/bin/env python
"""Map an ncu SASS source page (--page source --csv --print-source sass) of a
decode kernel onto CUDA source lines, using nvdisasm --print-line-info of the
same build, and print the source lines with the most stall samples.

    python tools/ncu_lines.py PROF_SASS.csv KERNEL.sass [kernel-substring] [top]
"""
import collections
import csv
import re
import sys


def line_map(sass_path, kname):
    """offset -> (file, line) for the function whose name contains kname."""
    cur, out, where = None, {}, None
    fn_re = re.compile(r"^\s*\.text\.(\S+):")
    li_re = re.compile(r'//## File "([^"]+)", line (\d+)')
    off_re = re.compile(r"/\*([0-9a-f]{4,})\*/")
    for ln in open(sass_path):
        m = fn_re.match(ln)
        if m:
            cur = m.group(1)
            continue
        if cur is None or kname not in cur:
            continue
        m = li_re.search(ln)
        if m:
            where = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = off_re.search(ln)
        if m and where:
            out[int(m.group(1), 16)] = where
    return out


def main():
    prof, sass = sys.argv[1], sys.argv[2]
    kname = sys.argv[3] if len(sys.argv) > 3 else "decode_kernel"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(prof)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    base = int(data[0][ix["Address"]], 16)
    lm = line_map(sass, kname)
    S, E = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    tot = 0
    for r in data:
        off = int(r[ix["Address"]], 16) - base
        key = lm.get(off, ("?", 0))
        smp = int(r[S] or 0)
        tot += smp
        a = agg[key]
        a[0] += smp
        a[1] += int(r[E] or 0)
        for c in stall_cols:
            v = int(r[ix[c]] or 0)
            if v:
                a[2][c] += v
    src = {}
    print(f"total samples {tot}, mapped offsets {len(lm)}")
    for key, (smp, ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        f, ln = key
        if f not in src:
            try:
                src[f] = open(f"csrc/{f}").read().split("\n")
            except OSError:
                src[f] = []
        text = src[f][ln - 1].strip()[:70] if 0 < ln <= len(src[f]) else ""
        tops = ", ".join(f"{k[6:]}:{v}" for k, v in st.most_common(2))
        print(f"{smp / tot * 100:5.1f}% {f}:{ln:<5} exec={ex:<9} {tops:40s} | {text}")


if __name__ == "__main__":
    main()
