mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_kernel -s 3 -c 1 -o gpurun_out/prof1 python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
