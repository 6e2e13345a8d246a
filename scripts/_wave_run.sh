export CUDA_DEVICE_MAX_CONNECTIONS=32
for i in 1 2; do for R in 1048576 1000000000000 262144; do echo "== single rows $R"
HBG_SINGLE_ROWS=$R HBG_GROW=legacy timeout 120 python scripts/prof_tree_shape.py 10500000 28 64 3 2>&1 | tail -1
HBG_SINGLE_ROWS=$R HBG_GROW=legacy timeout 120 python scripts/prof_tree_shape.py 10500000 28 16 3 2>&1 | tail -1
done; done
