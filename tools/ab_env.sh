#!/bin/bash
# A/B FFN tuning knobs: for each config in $CFGS and each env assignment list in $VARIANTS
# (';'-separated, e.g. "HEP_FFN_LIGHT=0 HEP_FFN_SWAP=0;HEP_FFN_LIGHT=1"), one short bench run.
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for c in ${CFGS:-dsv3 qwen3}; do
 for v in "${VS[@]}"; do
  env $v timeout 600 python bench.py --config $c --steps ${STEPS:-40} --warmup 5 --no-cpu-baseline --no-train 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$c [$v]', 'tok/s %.4g'%d['value'], 'ffn_ms %.3f'%d['stage_ms']['ffn'], 'TF/s %.0f'%r['achieved'], 'frac %.3f'%r['frac'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
 done
done
