"""Warp-stall samples and instructions of one kernel of an ncu report split
at its barriers (BAR.SYNC) -- which phase of a staged kernel costs what
(dev aid).  python scripts/ncu_segments.py rep.ncu-rep kernel_regex"""
import bisect, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = next(x for x in r if "Source" in x and "Address" in x)
rows = [x for x in r if x and x[0].startswith("0x")]
ia, isrc = h.index("Address"), h.index("Source")
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
prev, part = -1, []
for x in rows:
    a = int(x[ia], 16)
    if a < prev:
        break
    prev = a
    part.append(x)
base = int(part[0][ia], 16)
marks = [int(x[ia], 16) - base for x in part if "BAR.SYNC" in x[isrc] or "EXIT" in x[isrc]]
seg = {}
for x in part:
    k = bisect.bisect_right(marks, int(x[ia], 16) - base)
    s = seg.setdefault(k, [0, 0, None])
    s[0] += int(x[iss] or 0)
    s[1] += int(x[iex] or 0)
    if s[2] is None:
        s[2] = hex(int(x[ia], 16) - base)
tot = sum(v[0] for v in seg.values())
for k in sorted(seg):
    print(f"seg {k:2d} from {seg[k][2]:>7s}: samples {seg[k][0]:6d} ({100 * seg[k][0] / max(tot, 1):5.1f}%)  instr {seg[k][1]}")
