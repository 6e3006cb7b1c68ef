#!/bin/bash
# A/B of the epilogue warp count (column slices per TMEM lane quarter); rebuilds libhep.so per variant
for sp in ${SPLITS:-2 4}; do
  HEP_NVCC_DEFS="-DHEP_EPI_SPLIT=$sp" python -m paper_2511_16947_b200.build --force > /dev/null
  for c in ${CFGS:-qwen3 mixtral dsv3}; do
    for rep in 1 2; do
      python bench.py --config $c --steps 50 --no-cpu-baseline --no-train | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('split=$sp $c', round(d['value']), round(d['roofline']['achieved']), 'ffn_ms %.3f' % d['stage_ms']['ffn'], d['clocks']['sm_mhz'])"
    done
  done
done
python -m paper_2511_16947_b200.build --force > /dev/null
