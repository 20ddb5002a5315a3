#!/usr/bin/env python3
"""Map ncu per-SASS stall samples (ncu -i R --page source --csv) to source
lines using nvdisasm -g of the kernel's cubin.
    python tools/ncu_lines.py report.ncu-rep cubin mangled_substring"""
import collections, csv, re, subprocess, sys

rep, cubin, fn = sys.argv[1:4]
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(csvtxt.splitlines()))
h = r[1]
si = h.index('Warp Stall Sampling (All Samples)')
rows = [(int(x[0], 16), float(x[si] or 0)) for x in r[2:] if x and x[0].startswith('0x')]
base = min(a for a, _ in rows)
sass = subprocess.run(["nvdisasm", "-c", "-g", cubin], capture_output=True, text=True).stdout
off2 = {}
cur = None
infn = False
for ln in sass.split('\n'):
    if ln.startswith('.text.'):
        infn = fn in ln
        continue
    if not infn:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m:
        off2[int(m.group(1), 16)] = cur
agg = collections.Counter()
for a, v in rows:
    agg[off2.get(a - base)] += v
tot = sum(agg.values())
srcs = {}
for k, v in agg.most_common(25):
    if k is None:
        print(f"{100 * v / tot:5.1f}% ?"); continue
    f, l = k
    if f not in srcs:
        import glob
        p = glob.glob(f"/root/repo/**/{f}", recursive=True)
        srcs[f] = open(p[0]).read().split('\n') if p else []
    txt = srcs[f][l - 1].strip()[:90] if l <= len(srcs[f]) else ''
    print(f"{100 * v / tot:5.1f}% {f}:{l}: {txt}")
