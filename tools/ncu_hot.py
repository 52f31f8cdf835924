"""Top warp-stall-sampled SASS instructions of one kernel in an ncu report.
    python tools/ncu_hot.py <rep.ncu-rep> <kernel-regex> [launch-index] [top]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]


def num(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


rows = [r for r in rows if len(r) > 2 and r[0] != "Address"]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(num(r[si]) for r in rows if len(r) > si)
print(f"{lines[0][:120]}\ntotal samples {tot:.0f}")
ranked = sorted(rows, key=lambda r: -num(r[si]))[:top]
for r in ranked:
    s = num(r[si])
    reasons = sorted(((num(r[i]), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    rs = " ".join(f"{n}:{v/max(s,1)*100:.0f}%" for v, n in reasons if v > 0)
    print(f"{s/tot*100:5.1f}%  {r[0][-5:]}  {r[1].strip()[:60]:60s} {rs}")
