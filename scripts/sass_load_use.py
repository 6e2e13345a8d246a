"""Print, for each global load in a kernel, how many instructions later its
destination register is first read (a short distance = an exposed load latency)."""
import re
import subprocess
import sys

lib, pattern = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
for f in funcs:
    name = f.split("\n", 1)[0]
    if pattern not in name:
        continue
    ins = [m.group(1).strip() for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", f)]
    print("==", name[:100], len(ins), "instructions")
    for i, t in enumerate(ins):
        m = re.search(r"LDG\S*\s+(R\d+)", t)
        if not m:
            continue
        r = m.group(1)
        base = int(r[1:])
        width = 4 if ".128" in t else (2 if ".64" in t else 1)
        regs = {f"R{base + j}" for j in range(width)}
        for j in range(i + 1, min(i + 400, len(ins))):
            ops = re.findall(r"R\d+", ins[j].split(" ", 1)[-1])
            dst = ops[0] if ops and not ins[j].lstrip("@!P0123456789 ").startswith(("ST", "RED", "ATOM")) else None
            srcs = ops[1:] if dst else ops
            if regs & set(srcs):
                print(f"  {i:5d} {t[:60]:60s} first use +{j - i}: {ins[j][:60]}")
                break
