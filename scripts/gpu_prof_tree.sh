mkdir -p gpurun_out
for k in best_split hist_kernel partition_small; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 400 -c 1 -o gpurun_out/tree2_$k python scripts/prof_tree.py > gpurun_out/tree2_$k.log 2>&1
done
ls -la gpurun_out | grep tree2
