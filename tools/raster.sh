#!/bin/bash
for c in ${CFGS:-mixtral dsv3 qwen3}; do
 for gm in 0 2 4 8; do
  HEP_RASTER_GM=$gm timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --kernel-name-base demangled -k regex:"gemm2sm|gemm_kernel<.int.256" -c 2 --csv python bench.py --config $c --profile --steps 1 --warmup 1 --no-cpu-baseline --no-train 2>/dev/null | grep -E "dram__bytes_read|time_duration" | awk -F'","' -v c=$c -v p=$gm '{print c, "gm="p, $(NF-2), $NF}'
  HEP_RASTER_GM=$gm timeout 300 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --no-train 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c gm=$gm bench ffn_ms %.3f TF/s %.0f clk %s'%(d['stage_ms']['ffn'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
 done
done
