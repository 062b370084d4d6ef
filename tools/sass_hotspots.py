"""Attribute ncu SASS-level stall samples to CUDA source lines.
Usage: python tools/sass_hotspots.py <ncu-rep> <cubin> <kernel-substring> [top]
(needs -lineinfo; nvdisasm -g gives the address -> file:line map)"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def phase_of(src_lines):
    """PROF(n) markers of fused_small.cu -> [(first_line, n)] sorted."""
    marks = []
    for i, l in enumerate(src_lines, start=1):
        m = re.search(r"PROF\((\d+)\);", l)
        if m:
            marks.append((i, int(m.group(1))))
    return sorted(marks)


def main(rep, cubin, kname, top=40, src=None):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    cur, in_k, line_of = None, False, {}
    for l in dis.splitlines():
        if l.startswith("//----") and ".text." in l:
            in_k = kname in l
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and in_k:
            line_of[int(m.group(1), 16)] = cur
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    i0 = rows.index(hdr)
    ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    ir = [hdr.index(h) for h in reasons]
    data = []
    for r in rows[i0 + 1:]:
        if r and r[0] == "Address":
            break  # next kernel's section: only the first profiled kernel is attributed
        if len(r) == len(hdr):
            data.append(r)
    base = int(data[0][ia], 16)
    agg, tot = defaultdict(int), 0
    marks = phase_of(open(src).read().splitlines()) if src else []
    ph = defaultdict(lambda: defaultdict(int))
    for r in data:
        off = int(r[ia], 16) - base
        s = int(r[isamp] or 0)
        tot += s
        fl = line_of.get(off, ("?", 0))
        agg[fl] += s
        if marks and src and fl[0] == src.split("/")[-1]:
            prev = [n for (ln, n) in marks if ln <= fl[1]]
            key = f"after PROF({prev[-1]})" if prev else "setup"
        else:
            key = fl[0]
        for h, i in zip(reasons, ir):
            ph[key][h] += int(r[i] or 0)
    print(f"{tot} stall samples")
    for (f, ln), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * s / tot:6.2f} %  {f}:{ln}")
    if ph:
        print("\nstall samples by phase (top reasons):")
        for key, d in sorted(ph.items(), key=lambda kv: -sum(kv[1].values())):
            t = sum(d.values())
            best = sorted(d.items(), key=lambda kv: -kv[1])[:4]
            print(f"{100 * t / tot:6.2f} %  {key:16s} " + "  ".join(f"{k[6:]}={100 * v / max(t, 1):.0f}%" for k, v in best))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40,
         sys.argv[5] if len(sys.argv) > 5 else None)
