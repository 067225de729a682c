python -m pytest tests/test_gpu_parity.py tests/test_gpu_anytime.py tests/test_gpu_configs.py tests/test_dropin_cpp.py -x -q 2>&1 | tail -2
run() { echo "== $*"; env "$@" python tools/bench_configs.py --no-cpu --configs C1,C2,C3,C4,C5 --reps 2 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], '%.3e'%d['gpu_cells_per_s'], '%.3f ms'%d['gpu_ms'], 'e2e %.3e'%d['e2e_cells_per_s'])"; }
run MPGPU_COARSE=1
run MPGPU_COARSE=0
