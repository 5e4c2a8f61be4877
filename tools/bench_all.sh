#!/bin/bash
# bench lines for configs 3, 1, 2, 4, 0 + the reference arm + smoke() (run under gpurun):   ROUND=r2h bash tools/bench_all.sh
cd $GRAFT_REPO_ROOT
R=${ROUND:-r2h}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench3 rc=$?"
for c in 1 2 4 0; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --batched-config -1 --steps 5 --warmup 3 > gpurun_out/${R}_bench_config$c.json 2>> gpurun_out/${R}_bench.err; echo "bench$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_reference.json 2>> gpurun_out/${R}_bench.err; echo "ref rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
