export CUDA_DEVICE_MAX_CONNECTIONS=32
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('e2e', d['e2e']['ms_per_step'], 'pageable', d['e2e']['pageable_ms_per_step'], 'tree', d['tree']['sec_per_tree'], d['tree']['e2e_sec_per_tree'], d['tree']['e2e_pageable_sec_per_tree'])"
done
