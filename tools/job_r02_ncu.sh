# round-2 ncu evidence: one apply step's kernels (cfg3) and the Green's assemble kernel (cfg3)
python tools/profile_apply.py --applies 3 > gpurun_out/plain_apply.log 2>&1 && \
python tools/profile_greens.py --config 3 > gpurun_out/plain_greens.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stream_tma|contract_mma" -s 5 -c 5 \
    -o gpurun_out/r02_apply python tools/profile_apply.py --applies 3 > gpurun_out/ncu_apply.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:"assemble_kernel|spectra_|filter_design" -c 4 \
    -o gpurun_out/r02_greens python tools/profile_greens.py --config 3 > gpurun_out/ncu_greens.log 2>&1 ; \
ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/ncu_apply.log gpurun_out/ncu_greens.log
