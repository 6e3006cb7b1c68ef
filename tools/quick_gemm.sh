#!/bin/bash
# quick FFN check: GEMM parity, bench mixtral/dsv3 FFN stage, DRAM bytes per GEMM launch
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q --timeout 200 -x 2>&1 | tail -1
for c in ${CFGS:-mixtral dsv3}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c', 'tok/s %.4g'%d['value'], 'ffn_ms %.3f'%d['stage_ms']['ffn'], 'TF/s %.0f'%r['achieved'], 'frac_sus %.3f'%r['frac'], 'clk', d['clocks'])"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none \
    -k regex:"gemm_kernel<256" -c 2 --csv python bench.py --config $c --profile --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | grep gemm_kernel | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}'
done
