# A/B of hep_tuning.pair_wave_sync (minimum k-blocks per tile for the wave-synchronised
# producers of the CTA-pair GEMMs): time + energy per FFN, interleaved rounds
for c in mixtral dsv3; do
  timeout -s KILL 900 python tools/ffn_ab.py --config $c --variants "HEP_WAVE_SYNC=0;HEP_WAVE_SYNC=60" --iters 20 --rounds 12 >> gpurun_out/wave_ab3.txt 2>&1
done
