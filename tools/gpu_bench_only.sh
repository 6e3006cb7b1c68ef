#!/bin/bash
# The bench part of tools/gpu_measure.sh (default line, per-config lines, pipelined lines)
# plus the GPU tests, the router timeline / A/B and the reference arm.
set -x
R=${ROUND:-r02}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t_all_$R.log 2>&1
tail -2 gpurun_out/t_all_$R.log
timeout 900 python bench.py > gpurun_out/bench_default_$R.json 2> gpurun_out/bench_default_$R.err
for c in qwen3 dsv3; do
  timeout 900 python bench.py --config $c --other-configs "" > gpurun_out/bench_${c}_$R.json 2> gpurun_out/bench_${c}_$R.err
done
for c in qwen3 dsv3; do
  timeout 600 python bench.py --config $c --pipeline-ratio 0.5 --other-configs "" --no-cpu-baseline --no-train --no-balance-sweep > gpurun_out/bench_${c}_pipelined_$R.json 2>&1
done
timeout 200 python tools/router_stamps.py > gpurun_out/router_stamps_$R.txt 2>&1
timeout 300 python tools/router_ab.py --variants "router_pair=1;ws=1,router_pair=2;ws=1,router_pair=1" --graph --rounds 5 > gpurun_out/router_ab_$R.txt 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_mixtral_$R.json 2>&1
echo done
