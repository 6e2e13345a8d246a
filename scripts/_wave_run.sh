export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wave_grower or grow_tree or boosting" 2>&1 | tail -3
HBG_GROW_PROFILE=1 timeout 120 python scripts/prof_tree_shape.py 10500000 28 64 1 2>&1 | tail -4
HBG_GROW_PROFILE=1 timeout 120 python scripts/prof_tree_shape.py 1000000 28 64 1 2>&1 | tail -4
for R in 0 65536 262144 1048576; do for M in 8 16; do
  echo "== wave max $M spec rows $R"
  HBG_WAVE_SPEC_ROWS=$R HBG_WAVE_MAX=$M timeout 120 python scripts/prof_tree_shape.py 10500000 28 64 2 2>&1 | tail -1
  HBG_WAVE_SPEC_ROWS=$R HBG_WAVE_MAX=$M timeout 120 python scripts/prof_tree_shape.py 1000000 28 64 2 2>&1 | tail -1
done; done
