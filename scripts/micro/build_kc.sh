#!/bin/bash
# builds kc_bench (cluster panel vs column panel) and lat_bench next to their sources; extra nvcc flags pass through
set -e
D="$(cd "$(dirname "$0")" && pwd)"
C="$D/../../paper_1811_08057_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 "$D/lat_bench.cu" -o "$D/lat_bench"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo "$@" -I "$C" "$D/kc_bench.cu" "$C/k2_panel.cu" "$C/k2_cpanel.cu" -o "$D/kc_bench"
