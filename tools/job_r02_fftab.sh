#!/bin/bash
# A/B of the lateral passes' staging depth (stage timers of bench.py):
#   nstfy2  forward y pass with two 16 KB stages (three CTAs/SM)
#   fxreg1  forward x pass with r2 from per-thread loads (16 KB stage)
#   fxreg2  both forward passes double-staged, r2 per thread
#   nstinv2 inverse passes double-staged (two CTAs/SM)
mkdir -p gpurun_out
bash tools/ab_contraction.sh nstfy2=exp/nstfy2 fxreg1=exp/fxreg1 fxreg2=exp/fxreg2 nstinv2=exp/nstinv2 > gpurun_out/fftab1.log 2>&1
bash tools/ab_contraction.sh nstfy2=exp/nstfy2 fxreg1=exp/fxreg1 fxreg2=exp/fxreg2 nstinv2=exp/nstinv2 > gpurun_out/fftab2.log 2>&1
for v in fxreg2 nstinv2; do
  EMIE_CU_LIBRARY=exp/$v/libemie_cu.so timeout 600 python -m pytest tests/test_gpu_sizes.py tests/test_gpu_e2e_parity.py -q -x > gpurun_out/fftab_tests_$v.log 2>&1
  echo "$v tests rc=$?" >> gpurun_out/fftab1.log
done
cat gpurun_out/fftab1.log gpurun_out/fftab2.log
