mkdir -p gpurun_out
for k in best_split partition_small hist_kernel; do
timeout 300 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:$k -s 150 -c 1 -o gpurun_out/tree3_$k python scripts/prof_tree.py 2000000 1 > gpurun_out/tree3_$k.log 2>&1
done
ls -la gpurun_out | grep tree3
