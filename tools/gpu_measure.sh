#!/bin/bash
# One measurement round on the B200 box: tests, ncu launch lists (-> per-launch DRAM
# traffic), bench (3 configs + pipelined variant + reference arm), full ncu captures
# of the top kernels.  Output under gpurun_out/ (copy what is judged to profiles/).
set -x
R=${ROUND:-r02}
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t_all_$R.log 2>&1
tail -2 gpurun_out/t_all_$R.log
timeout 120 python tools/sched_timing.py > gpurun_out/sched_timing_$R.json 2>&1
for c in mixtral qwen3 dsv3; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -k regex:"hep::|gemm::|sched_kernel|permute|combine|chunk|plan_prep|gate_topk" -c 17 --csv \
    --log-file gpurun_out/launches_${c}_$R.csv python bench.py --config $c --profile --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
# the launch lists are committed under profiles/<round>/ afterwards: record that path
python tools/traffic.py --tracked=profiles/${R%?} gpurun_out/launches_mixtral_$R.csv gpurun_out/launches_qwen3_$R.csv gpurun_out/launches_dsv3_$R.csv > gpurun_out/traffic_$R.json
cp gpurun_out/traffic_$R.json profiles/traffic.json
# the default line (Mixtral + Qwen3 / DSv3 folded in), then each config as the primary
timeout 900 python bench.py > gpurun_out/bench_default_$R.json 2> gpurun_out/bench_default_$R.err
for c in qwen3 dsv3; do
  timeout 900 python bench.py --config $c --other-configs "" > gpurun_out/bench_${c}_$R.json 2> gpurun_out/bench_${c}_$R.err
done
for c in qwen3 dsv3; do
  timeout 600 python bench.py --config $c --pipeline-ratio 0.5 --other-configs "" --no-cpu-baseline --no-train --no-balance-sweep > gpurun_out/bench_${c}_pipelined_$R.json 2>&1
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_mixtral_$R.json 2>&1
timeout 300 python tools/lp_timing.py > gpurun_out/lp_timing_$R.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm2sm_kernel|gemm_kernel|sched_kernel|permute|combine|chunk_map|plan_prep" -c 9 \
  -o gpurun_out/prof_mixtral_$R python bench.py --config mixtral --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_mixtral_$R.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm2sm_kernel|gemm_kernel<.int.256|sched_kernel|permute|combine" -c 8 \
  -o gpurun_out/prof_dsv3_$R python bench.py --config dsv3 --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_dsv3_$R.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm2sm_kernel" -c 2 \
  -o gpurun_out/prof_qwen3_$R python bench.py --config qwen3 --profile --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_qwen3_$R.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm2sm_kernel" --launch-skip 6 -c 6 \
  -o gpurun_out/prof_train_qwen3_$R python tools/train_step.py --config qwen3 --iters 2 > gpurun_out/ncu_train_qwen3_$R.log 2>&1
# K1 router+gate: back-to-back A/B inside CUDA graphs (memset vs in-kernel histogram zeroing,
# 1-CTA vs CTA pairs), per-CTA timeline (diagnostics build, tools/build_diag.sh), and one full
# ncu capture per shape
timeout 300 python tools/router_ab.py --variants "router_pair=1,router_pair=2,ws=1" --graph --rounds 5 > gpurun_out/router_ab_$R.txt 2>&1
timeout 200 python tools/router_stamps.py > gpurun_out/router_stamps_$R.txt 2>&1
for c in mixtral qwen3 dsv3; do
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm" \
    --launch-skip 3 -c 1 -o gpurun_out/prof_router_${c}_$R python tools/router_one.py $c 5 > /dev/null 2>&1
done
# summarise the full captures on the box (copy-back is capped at 64 MiB) and drop the reports
for r in gpurun_out/prof_*_$R.ncu-rep; do
  python tools/ncu_summary.py $r > ${r%.ncu-rep}.md 2>&1
done
python tools/ncu_hot.py gpurun_out/prof_qwen3_$R.ncu-rep gemm2sm 30 1 > gpurun_out/hot_qwen3_gemm2_$R.txt 2>&1
python tools/ncu_hot.py gpurun_out/prof_train_qwen3_$R.ncu-rep gemm2sm 30 2 > gpurun_out/hot_train_qwen3_dgrad_$R.txt 2>&1
python tools/ncu_hot.py gpurun_out/prof_router_dsv3_$R.ncu-rep gemm 30 > gpurun_out/hot_router_dsv3_$R.txt 2>&1
rm -f gpurun_out/prof_*_$R.ncu-rep
echo done
