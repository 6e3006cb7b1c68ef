#!/bin/bash
# Build the router-timeline diagnostics library (libhep_diag.so, -DHEP_ROUTER_STAMPS) next
# to the product libhep.so, then rebuild the product library.
set -e
cd "$(dirname "$0")/.."
touch paper_2511_16947_b200/csrc/gemm_sm100.cu
HEP_NVCC_DEFS=-DHEP_ROUTER_STAMPS python -m paper_2511_16947_b200.build >/dev/null
cp paper_2511_16947_b200/libhep.so paper_2511_16947_b200/libhep_diag.so
touch paper_2511_16947_b200/csrc/gemm_sm100.cu
python -m paper_2511_16947_b200.build >/dev/null
nm -D paper_2511_16947_b200/libhep_diag.so | grep -q hep_diag_router_stamps && echo diag ok
