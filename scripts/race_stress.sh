#!/bin/bash
# Race stress in place of compute-sanitizer (closed on this pool): rebuild the library with
# MCND_JITTER=1 (pseudo-random sleeps at every inter-CTA hand-off of K1 and the panel kernel:
# before publishing a record / pivot row, before releasing a flag, before polling, before the
# bulk updates), run the protocol-sensitive parity tests (bitwise vs the reference, the
# emulated multi-GPU push protocol, the two blocked schedules against each other, the headline
# C3 golden, the native multi-GPU driver), then restore the normal build.
set -u
cd "$(dirname "$0")/.."
out=${1:-gpurun_out/r2_race_stress.log}
MCND_BUILD_DEFINES="MCND_JITTER=1" python -c "from paper_1811_08057_b200.build import build; build(force=True)"
echo "NANOSLEEP instructions, jitter build: $(cuobjdump -sass paper_1811_08057_b200/lib/libmcnd_b200.so | grep -c NANOSLEEP)" > "$out.sass"
python -m pytest tests/test_gpu_parity.py tests/test_gpu_mg.py -m gpu -q -p no:cacheprovider \
  -k "serial_bitwise or mc_parallel_bitwise or emulated_ranks or kernel_shapes or blocked_lookahead or blocked_c3 or blocked_vs_oracle or panel_kernels_agree or singular or native_driver or ge_logdet" \
  > "$out" 2>&1
rc=$?
echo "jitter build exit $rc" >> "$out"
python -c "from paper_1811_08057_b200.build import build; build(force=True)"
echo "NANOSLEEP instructions, normal build: $(cuobjdump -sass paper_1811_08057_b200/lib/libmcnd_b200.so | grep -c NANOSLEEP)" >> "$out.sass"
cat "$out.sass" >> "$out"
exit $rc
