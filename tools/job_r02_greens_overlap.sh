#!/bin/bash
# A/B: Green's split build with the image kernel of batch i+1 overlapped with
# the pair kernel of batch i on a second stream (default) vs serial
mkdir -p gpurun_out
{
for c in 3 4; do
  reps=4; [ $c = 4 ] && reps=2
  echo "== cfg$c overlap (1 GB buffers x2)"; python tools/time_greens.py --config $c --reps $reps
  echo "== cfg$c overlap, 2 GB buffers x2"; EMIE_CU_GREENS_IMG_MB=4096 python tools/time_greens.py --config $c --reps $reps
  echo "== cfg$c serial"; EMIE_CU_GREENS_OVERLAP=0 python tools/time_greens.py --config $c --reps $reps
done
} > gpurun_out/greens_overlap.log 2>&1
timeout 900 python -m pytest tests/test_gpu_greens.py tests/test_gpu_greens_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/greens_overlap_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/greens_overlap.log
tail -3 gpurun_out/greens_overlap_tests.log >> gpurun_out/greens_overlap.log
cat gpurun_out/greens_overlap.log
