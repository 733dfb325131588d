"""Summarise an ncu --page source --print-source sass CSV: instruction totals by block of equal
execution count, with warp-stall samples.  usage: python tools/sass_hot.py file.csv [n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n_show = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]; data = rows[2:]
iA, iS, iSamp, iEx = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"))
base = int(data[0][iA], 16)
tot = sum(int(r[iEx]) for r in data); ts = sum(int(r[iSamp]) for r in data)
print("total inst", tot, "samples", ts)
blocks = []
for r in data:
    off = int(r[iA], 16) - base; ex = int(r[iEx]); sm = int(r[iSamp])
    if blocks and blocks[-1][2] == ex and off - blocks[-1][1] == 16:
        b = blocks[-1]; b[1] = off; b[3] += ex; b[4] += sm; b[5] += 1; b[6].append(r[iS].strip().split()[0] if r[iS].strip() else "")
    else:
        blocks.append([off, off, ex, ex, sm, 1, [r[iS].strip().split()[0] if r[iS].strip() else ""]])
blocks.sort(key=lambda b: -b[3])
for b in blocks[:n_show]:
    ops = " ".join(sorted(set(o.split(".")[0] for o in b[6])))[:60]
    print(f"0x{b[0]:05x}-0x{b[1]:05x} count {b[2]:>11} n {b[5]:4d} inst {b[3]/tot*100:5.1f}% samp {b[4]/ts*100:5.1f}% {ops}")
