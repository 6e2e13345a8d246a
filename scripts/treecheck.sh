mkdir -p gpurun_out
for cfg in "X=1" "HBG_NO_PDL=1"; do
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/tc.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/tc.json').read().strip().splitlines()[-1]); t=d['tree']; print('$cfg', t['sec_per_tree'], t['e2e_sec_per_tree'], t['hist_kernel_ms_per_tree'])"
done
HBG_GROW_PROFILE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-variants --no-cpu-baseline 2> gpurun_out/tc_prof.err > /dev/null; tail -30 gpurun_out/tc_prof.err
