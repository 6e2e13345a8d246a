#!/bin/bash
# A/B of the pad-free histogram kernel (hist_dup.cu) against the 32-step one
# on the bench workload; parity of the d=28 cases first.
mkdir -p gpurun_out
TAG=${1:-dup}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host_dropin or full_size or edge or deterministic or identity or subtraction or row_indexed or contiguous or golden_histograms" > gpurun_out/${TAG}_parity.txt 2>&1
tail -3 gpurun_out/${TAG}_parity.txt
for cfg in "HBG_HIST_DUP=0" "HBG_DUP_R=1" "HBG_DUP_R=2" "HBG_DUP_R=3"; do
  env $cfg timeout 300 python bench.py --steps 100 --warmup 5 --no-variants --no-cpu-baseline --no-tree > gpurun_out/${TAG}_bench_${cfg}.json 2>/dev/null
  python - "$cfg" gpurun_out/${TAG}_bench_${cfg}.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
r=d["roofline"]
print(f"{sys.argv[1]:16s} step {d['ms_per_step']*1e3:7.1f} us  kernel {r['kernel_ms']*1e3:7.1f} us  frac {r['frac']:.4f}")
PY
done
