#!/bin/bash
# compute-sanitizer over scripts/sanitize_run.py (every device kernel at small
# sizes): memcheck, racecheck, synccheck, initcheck.  Logs under gpurun_out/,
# one summary line per tool on stdout.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --num-cuda-barriers 256 --print-limit 100000 python scripts/sanitize_run.py > gpurun_out/sanitize_$t.txt 2>&1
  echo "$t rc=$? $(grep -cE '^ok ' gpurun_out/sanitize_$t.txt) steps: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$t.txt | tail -1)"
done
