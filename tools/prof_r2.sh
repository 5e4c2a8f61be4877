#!/bin/bash
# round-2 evidence: bench lines (config 3 default + configs 0/1/2/4 + reference arm),
# ncu launch list of config 3, DRAM bytes per pass for every config, one --set full
# capture of config 3's two passes.   ROUND=r2b bash tools/prof_round.sh ... (run under gpurun)
cd $GRAFT_REPO_ROOT
R=${ROUND:-r2b}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench3 rc=$?"
for c in 1 2 4 0; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --batched-config -1 --steps ${STEPS:-5} --warmup 3 > gpurun_out/${R}_bench_config$c.json 2>> gpurun_out/${R}_bench.err; echo "bench$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_reference.json 2>> gpurun_out/${R}_bench.err; echo "ref rc=$?"
for c in 3 1 2 4 0; do
  timeout 900 python bench.py --profile-only --config $c > /dev/null 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"k_pa|k_plane|k_fx|k_ex|k_y3" -s 20 -c 6 --csv --log-file gpurun_out/${R}_dram_config$c.csv \
      python bench.py --profile-only --config $c > /dev/null 2>&1; echo "dram$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
    --log-file gpurun_out/${R}_launches_config3.csv python bench.py --profile-only --config 3 > /dev/null 2>&1; echo "list rc=$?"
if [ -z "$NOFULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pa|k_plane" -s 10 -c 2 \
    -o gpurun_out/full_${R}_c3 python bench.py --profile-only --config 3 > gpurun_out/${R}_ncu_full.log 2>&1; echo "full rc=$?"
fi
