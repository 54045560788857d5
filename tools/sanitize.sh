#!/bin/bash
# compute-sanitizer over the hand-synchronised kernels (tools/sanitize_driver.py).
# usage: tools/sanitize.sh TOOL [CASE...]   (TOOL: racecheck | synccheck | memcheck)
# Writes gpurun_out/sanitize_<tool>_<case>.log; each case under its own timeout.
tool=${1:-racecheck}; shift
cases=${@:-qrcp_cluster qrcp_grid qrcp_general saso trsm potrf gram cond all_small}
mkdir -p gpurun_out
for c in $cases; do
  env_extra=""
  [ "$c" = "qrcp_grid" ] && env_extra="CQRRPT_QRCP_NOCLUSTER=1"
  [ "$c" = "qrcp_general" ] && env_extra="CQRRPT_QRCP_GENERAL=1"
  log=gpurun_out/sanitize_${tool}_${c}.log
  echo "== $tool $c ($env_extra)" > $log
  env $env_extra timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 \
      python tools/sanitize_driver.py $c >> $log 2>&1
  echo "exit=$?" >> $log
  tail -3 $log
done
