export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wave_grower or grow_tree or boosting" 2>&1 | tail -1
for i in 1 2; do
echo "== old"; HBG_PKG_ROOT=$PWD/_ab_old timeout 120 python scripts/prof_tree_shape.py 10500000 28 16 3 2>&1 | tail -1
echo "== new"; timeout 120 python scripts/prof_tree_shape.py 10500000 28 16 3 2>&1 | tail -1
done
echo "== new k64"; timeout 120 python scripts/prof_tree_shape.py 10500000 28 64 3 2>&1 | tail -1
echo "== new 1M"; timeout 120 python scripts/prof_tree_shape.py 1000000 28 64 3 2>&1 | tail -1
