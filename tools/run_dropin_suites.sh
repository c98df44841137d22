#!/bin/bash
# The reference's own suites (greens, layered, hankel, quad, toeplitz; unchanged, compiled against
# the B200 drop-in by `make -C oracle dropin`), one test case at a time with a
# time limit each; per-case status and wall time into gpurun_out/dropin_suites.log
out=gpurun_out/dropin_suites.log
mkdir -p gpurun_out; : > $out
run() {  # binary, case-name substring
  local t0=$(date +%s)
  timeout ${3:-900} $1 -tc="$2" > /tmp/tc.out 2> /tmp/tc.err
  local rc=$?
  local t1=$(date +%s)
  printf "%-20s rc=%-3s %5ss  %s :: %s\n" "$(basename $1)" $rc $((t1 - t0)) "$(grep -h 'test cases' /tmp/tc.out)" "$2" >> $out
  grep -h -m8 "FAILED" /tmp/tc.err >> $out
}
# the brute-force spectral-integration case of test_greens.cpp (~13 min through
# per-point device calls) only with FULL=1
while IFS= read -r tc; do
  [ "$tc" = "cross couplings match direct spectral integration" ] && [ "${FULL:-0}" != 1 ] && continue
  run oracle/_ref/dropin_test_greens "$tc"
done < tools/dropin_cases_greens.txt
while IFS= read -r tc; do run oracle/_ref/dropin_test_layered "$tc"; done < tools/dropin_cases_layered.txt
while IFS= read -r tc; do run oracle/_ref/dropin_test_hankel "$tc"; done < tools/dropin_cases_hankel.txt
run oracle/_ref/dropin_test_quad ""
run oracle/_ref/dropin_test_toeplitz ""
cat $out
