#!/bin/bash
# Round measurement: bench (default args), the ncu launch list of a short bench
# command, and one full ncu capture of the bench's cell-map kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
SHORT="python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu --no-c3 --no-c5"
timeout 300 $SHORT > gpurun_out/bench_short.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launches.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cellmap -s 3 -c 1 -o gpurun_out/prof_bench $SHORT > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
