# Round profiles (run under gpurun): default bench line (C3 + C5 sub-record + CPU baseline), the
# C5 launch list, ncu --set full of one large persistent K = 256 group GEMM launch in C5.
set -x
mkdir -p gpurun_out
if [ "${SKIP_BENCH:-0}" = 0 ]; then
timeout 900 python bench.py > gpurun_out/r2b_bench_default.json 2> gpurun_out/r2b_bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_c5.csv \
    python scripts/k2_prof.py 32768 > gpurun_out/r2b_launches_c5.log 2>&1
fi
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k 'regex:w4_kernel<.int.256, .int.3, .int.2, .int.16, .int.2>' --launch-skip 4 --launch-count 1 \
    -o gpurun_out/r2b_ncu_gemm256_c5 -f python scripts/k2_prof.py 32768 > gpurun_out/r2b_ncu_gemm256.log 2>&1
tail -3 gpurun_out/r2b_ncu_gemm256.log
