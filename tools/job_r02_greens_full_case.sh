# the brute-force case of the reference's test_greens.cpp ("cross couplings match direct spectral
# integration", ~13 min through per-point device calls) against the drop-in on one B200
cd $GRAFT_REPO_ROOT
t0=$(date +%s)
timeout 2400 oracle/_ref/dropin_test_greens -tc="cross couplings match direct spectral integration" > gpurun_out/greens_full_case.out 2> gpurun_out/greens_full_case.err
rc=$?
t1=$(date +%s)
printf "dropin_test_greens   rc=%-3s %5ss  %s :: cross couplings match direct spectral integration (FULL=1)\n" $rc $((t1 - t0)) "$(grep -h 'test cases' gpurun_out/greens_full_case.out)" | tee gpurun_out/greens_full_case.log
grep -h -m8 "FAILED" gpurun_out/greens_full_case.err gpurun_out/greens_full_case.out | tee -a gpurun_out/greens_full_case.log
