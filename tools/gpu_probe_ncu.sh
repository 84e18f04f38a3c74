cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/cellmap_probe 1024 > gpurun_out/probe_plain.jsonl 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cellmap -s 6 -c 1 -o gpurun_out/prof_probe_mode1 ./tools/cellmap_probe 1024 > gpurun_out/ncu_probe1.log 2>&1
