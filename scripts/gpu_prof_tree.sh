mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:best_split -s 300 -c 2 -o gpurun_out/tree_split python scripts/prof_tree.py > gpurun_out/tree_split.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hist_kernel -s 300 -c 2 -o gpurun_out/tree_hist python scripts/prof_tree.py > gpurun_out/tree_hist.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:partition_count -s 300 -c 1 -o gpurun_out/tree_part python scripts/prof_tree.py > gpurun_out/tree_part.log 2>&1
tail -2 gpurun_out/tree_*.log
