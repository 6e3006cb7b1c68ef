V="HEP_WAVE_SYNC=0;HEP_WAVE_SYNC=1;HEP_WAVE_SYNC=0;HEP_WAVE_SYNC=1"
timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --kernel-name regex:gemm2sm --clock-control none --csv --log-file gpurun_out/traffic_ab_mixtral.csv python tools/ffn_ab.py --config mixtral --variants "$V" --iters 1 --rounds 1 > gpurun_out/traffic_ab_mixtral.log 2>&1
timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --kernel-name regex:gemm2sm --clock-control none --csv --log-file gpurun_out/traffic_ab_qwen3.csv python tools/ffn_ab.py --config qwen3 --variants "$V" --iters 1 --rounds 1 > gpurun_out/traffic_ab_qwen3.log 2>&1
for c in mixtral qwen3 dsv3; do
  timeout -s KILL 600 python tools/ffn_ab.py --config $c --variants "HEP_WAVE_SYNC=0;HEP_WAVE_SYNC=1" --iters 20 --rounds 6 >> gpurun_out/wave_ab.txt 2>&1
done
