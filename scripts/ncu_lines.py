"""Warp-stall samples per CUDA source line of one ncu report:
    python scripts/ncu_lines.py REP [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(io.StringIO(out)))
f, hits = None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "Function Name") or not r[0]:
        continue
    try:
        hits.append((int(float(r[4])), f, int(r[0]), r[1]))
    except (ValueError, IndexError):
        pass
tot = sum(h[0] for h in hits) or 1
print(f"total samples {tot}")
for v, fn, ln, s in sorted(hits, reverse=True)[:top]:
    print(f"{v:8d} {100 * v / tot:5.1f}%  {fn}:{ln:<5d} {s.strip()[:90]}")
