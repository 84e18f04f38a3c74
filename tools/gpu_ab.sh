#!/bin/bash
# A/B timing of library variants on one box: tools/gpu_ab.sh default nowres ...
# ("default" = the in-tree build; others = build_var/<name>/libhermb200.so).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
out=gpurun_out/ab.txt
rm -f $out
CONFIGS=${AB_CONFIGS:-"diss:2:1024 diss:3:1024 diss:4:1024 diss:5:1024 diss:6:1024 diss:7:1024 diss:8:1024 cons:3:2048:walls cons:4:2048:walls cons:5:2048:walls cons:8:2048:walls"}
# parity of each variant first (a broken variant's timing means nothing)
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=build_var/$v/libhermb200.so; fi
  echo "parity [$v]: $(HERMB200_LIB=$lib timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_interior.py -q -x 2>&1 | tail -1)" >> $out
done
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then lib=""; else lib=build_var/$v/libhermb200.so; fi
    for c in $CONFIGS; do
      IFS=: read -r sch m n walls <<< "$c"
      HERMB200_LIB=$lib timeout 120 python tools/prof_step.py --scheme $sch --m $m --n $n ${walls:+--walls} --tag "$v/" >> $out 2>&1
    done
  done
done
