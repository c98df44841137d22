# A/B: spectra on the TMA engine vs the per-CTA kernels (Green's build stage
# timers), and 4 CTAs/SM for the forward y pass (apply stage timers)
python tools/time_greens.py --config 3 --reps 3 > gpurun_out/ab_spectra_tma.log 2>&1
EMIE_CU_SPECTRA_NO_TMA=1 python tools/time_greens.py --config 3 --reps 3 > gpurun_out/ab_spectra_old.log 2>&1
python tools/time_greens.py --config 4 --reps 2 >> gpurun_out/ab_spectra_tma.log 2>&1
EMIE_CU_SPECTRA_NO_TMA=1 python tools/time_greens.py --config 4 --reps 2 >> gpurun_out/ab_spectra_old.log 2>&1
python -m pytest tests/test_gpu_sizes.py tests/test_gpu_e2e_parity.py -q -k "sizes or cfg3" > gpurun_out/ab_tests.log 2>&1
bash tools/ab_contraction.sh minb4=exp/minb4 > gpurun_out/ab_minb4.log 2>&1
tail -4 gpurun_out/ab_spectra_tma.log gpurun_out/ab_spectra_old.log; tail -3 gpurun_out/ab_tests.log; cat gpurun_out/ab_minb4.log
