#!/bin/bash
# round-end evidence: bench lines (configs 1, 0, 2, 3, 4 + reference arm), ncu launch list and one full capture
cd $GRAFT_REPO_ROOT
R=${ROUND:-r1g}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench1 rc=$?"
for c in 0 2 3 4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_bench_config$c.json 2>> gpurun_out/${R}_bench.err; echo "bench$c rc=$?"; done
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_reference.json 2>> gpurun_out/${R}_bench.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_config1.csv python bench.py --profile-only > gpurun_out/${R}_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pa|k_plane" -s 10 -c 2 -o gpurun_out/full_${R} python bench.py --profile-only > gpurun_out/${R}_ncu_full.log 2>&1; echo "ncu full rc=$?"
