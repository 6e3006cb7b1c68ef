#!/bin/bash
# A/B the TMA L2 policies of the FFN GEMMs: pol = A | B<<2 (1 normal, 2 last, 3 first); 0 = defaults
for c in ${CFGS:-mixtral dsv3}; do
 for pol in 0 5 13 7 10; do
  HEP_L2POL=$pol timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --kernel-name-base demangled -k regex:"gemm2sm|gemm_kernel<.int.256" -c 2 --csv python bench.py --config $c --profile --steps 1 --warmup 1 --no-cpu-baseline --no-train 2>/dev/null | grep -E "dram__bytes_read|time_duration" | awk -F'","' -v c=$c -v p=$pol '{print c, "pol="p, $(NF-2), $NF}'
  HEP_L2POL=$pol timeout 300 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --no-train 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c pol=$pol bench ffn_ms %.3f TF/s %.0f clk %s'%(d['stage_ms']['ffn'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
 done
done
