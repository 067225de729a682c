#!/bin/bash
# quick C4 timing of one or more library builds: tools/quick_bench.sh lib1.so [lib2.so ...]
for L in "$@"; do
  MPGPU_LIB=$(realpath $L) python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$L value %.4e frac %.3f join_ms %.1f'%(d['value'],d['roofline']['frac'],d['roofline']['join_ms_per_launch']))"
done
