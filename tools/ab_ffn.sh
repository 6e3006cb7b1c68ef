#!/bin/bash
# A/B the FFN kernel variants (1-CTA vs CTA-pair) on the bench configs
for c in ${CFGS:-mixtral qwen3 dsv3}; do
 for pair in 0 1; do
  HEP_FFN_PAIR=$pair timeout 600 python bench.py --config $c --steps ${STEPS:-60} --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$c pair=$pair', 'tok/s %.4g'%d['value'], 'ffn_ms %.3f'%d['stage_ms']['ffn'], 'TF/s %.0f'%r['achieved'], 'frac_sus %.3f'%r['frac'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
 done
done
