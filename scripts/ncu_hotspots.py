"""Per-region warp-stall samples of one kernel in an ncu report (source page, SASS).
    python scripts/ncu_hotspots.py REP [kernel-regex] [chunk]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "hist_kernel"
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 48
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hi = his[0]
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
end = his[1] - 1 if len(his) > 1 else len(rows)
data = [r for r in rows[hi + 1:end] if len(r) == len(hdr)]


def v(r, k="Warp Stall Sampling (All Samples)"):
    try:
        return int(r[ix[k]] or 0)
    except ValueError:
        return 0


tot = sum(v(r) for r in data)
print(f"{rows[hi-1][1][:90]}\ntotal samples {tot}, {len(data)} SASS instructions")
for c in range(0, len(data), chunk):
    s = sum(v(r) for r in data[c:c + chunk])
    if s >= tot * 0.03:
        top = max(data[c:c + chunk], key=v)
        print(f"  [{c:5d}+{chunk}] {s:6d} ({100*s/tot:4.1f}%)  hottest: {v(top):5d} {top[ix['Source']].strip()[:60]}")
