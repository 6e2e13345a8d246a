export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wave_grower or grow_tree or boosting" 2>&1 | tail -2
HBG_GROW_PROFILE=1 timeout 120 python scripts/prof_tree_shape.py 1000000 28 64 1 2>&1 | tail -5
timeout 120 python scripts/prof_tree_shape.py 1000000 28 64 3 2>&1 | tail -1
HBG_GROW=wave timeout 120 python scripts/prof_tree_shape.py 10500000 28 64 3 2>&1 | tail -1
timeout 120 python scripts/prof_tree_shape.py 10500000 28 64 3 2>&1 | tail -1
