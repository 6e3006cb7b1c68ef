mkdir -p gpurun_out
timeout 300 python tools/sched_timing.py --variants "$VARS" > gpurun_out/sched_ab_$R.txt 2>&1
python - <<'PY'
import json,os
txt=open(f"gpurun_out/sched_ab_{os.environ['R']}.txt").read()
dec=json.JSONDecoder(); i=0
while True:
    j=txt.find("{",i)
    if j<0: break
    try: o,k=dec.raw_decode(txt[j:])
    except Exception as ex: print(txt[j:j+2000]); break
    i=j+k
    print(o["variant"], {c:(o[c]["lexmin"],o[c]["route"],o[c]["total_cycles"],round(o[c]["us_per_launch_back_to_back"],1),o[c]["same_as_default"]) for c in ("mixtral","qwen3","dsv3")})
PY
timeout 900 python -m pytest tests/test_sched_gpu.py tests/test_sched_props_gpu.py tests/test_stress_gpu.py tests/test_layer_gpu.py tests/test_lp_gpu.py -m gpu -q -x --timeout 800 > gpurun_out/t_sched_$R.log 2>&1; tail -5 gpurun_out/t_sched_$R.log
