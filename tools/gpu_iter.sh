#!/bin/bash
# One GPU iteration: parity tests, a short bench, an ncu capture of k_join.
# usage: tools/gpu_iter.sh TAG [ncu]
TAG=${1:-iter}
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]);print('value %.4e frac %.3f ms %.1f clk %s'%(d['value'],d['roofline']['frac'],d['ms_per_step'],d['clocks']))"
if [ "$2" == "ncu" ]; then
  python tools/profile_step.py --config C4 > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_join --launch-skip 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py --config C4 > gpurun_out/ncu_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_$TAG.log
fi
