#!/bin/bash
# per-GEMM raster band sweep: DRAM bytes + time of the two FFN GEMMs (ncu) and the bench FFN TF/s
for c in ${CFGS:-mixtral}; do
 for g1 in ${GM1S:-6 8 12}; do for g2 in ${GM2S:-4 8}; do
  export HEP_RASTER_GM1=$g1 HEP_RASTER_GM2=$g2
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --kernel-name-base demangled -k regex:"gemm2sm|gemm_kernel<.int.256" -c 2 --csv python bench.py --config $c --profile --steps 1 --warmup 1 --no-cpu-baseline --no-train 2>/dev/null | grep -E "dram__bytes_read|time_duration" | awk -F'","' -v c=$c -v p="$g1/$g2" '{print c, "gm="p, $(NF-2), $NF}'
  timeout 300 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --no-train 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c gm=$g1/$g2 bench ffn_ms %.3f TF/s %.0f clk %s'%(d['stage_ms']['ffn'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
 done; done
done
