#!/bin/bash
# compute-sanitizer evidence for the cell-map kernel: one tool per
# call, small grids, PDL and the dynamic tile schedule as built.
#   gpurun -- 'bash tools/gpu_sanitize.sh racecheck'   (or synccheck, memcheck, initcheck)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
tool=${1:-racecheck}
mkdir -p gpurun_out
out=gpurun_out/sanitize_$tool.txt
: > $out
CONFIGS=${SAN_CONFIGS:-"diss:4:256 diss:4:96 cons:5:256:walls cons:5:64:walls diss:2:256 diss:3:256 diss:6:128 cons:4:128:walls"}
for c in $CONFIGS; do
  IFS=: read -r sch m n walls <<< "$c"
  echo "=== $tool: $sch m=$m n=$n ${walls}" >> $out
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
    python tools/prof_step.py --scheme $sch --m $m --n $n ${walls:+--walls} --steps 4 --reps 1 >> $out 2>&1
  echo "rc=$?" >> $out
done
grep -E "^===|ERROR SUMMARY|RACECHECK SUMMARY|rc=" $out > gpurun_out/sanitize_${tool}_summary.txt
