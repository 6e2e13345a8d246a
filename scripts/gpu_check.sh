#!/bin/bash
# One GPU round trip: GPU tests, the bench line, the launch list and one ncu
# --set full capture of the histogram kernel. Usage: bash scripts/gpu_check.sh TAG [pytest args]
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest.txt 2>&1
  tail -15 gpurun_out/${TAG}_pytest.txt
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
     python bench.py --steps 5 --warmup 3 --no-variants --no-cpu-baseline ${BENCH_ARGS:-} > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_kernel -s 3 -c 1 \
     -o gpurun_out/${TAG}_prof python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline ${BENCH_ARGS:-} \
     > gpurun_out/${TAG}_ncu.log 2>&1
  tail -2 gpurun_out/${TAG}_ncu.log
fi
