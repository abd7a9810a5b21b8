# Round profiles with the cluster panel kernel (run under gpurun): bench lines, the C3 launch
# list, ncu --set full of one cluster panel pair launch inside a C3 call, the C3 timeline.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2c_bench_default.json 2> gpurun_out/r2c_bench_default.err
for c in c1 c2 c4; do timeout 300 python bench.py --config $c > gpurun_out/r2c_bench_$c.json 2> gpurun_out/r2c_bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2c_bench_reference.json 2> gpurun_out/r2c_bench_reference.err
MCND_DEBUG_TIMELINE=1 timeout 300 python scripts/k2_timeline.py 8000 > gpurun_out/r2c_k2_timeline_c3.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches_c3.csv \
    python scripts/k2_c3_prof.py > gpurun_out/r2c_launches_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k 'regex:kc_panel_kernel' --launch-skip 70 --launch-count 1 \
    -o gpurun_out/r2c_ncu_kc_c3 -f python scripts/k2_c3_prof.py > gpurun_out/r2c_ncu_kc.log 2>&1
tail -3 gpurun_out/r2c_ncu_kc.log
