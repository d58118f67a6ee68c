python -m pytest tests/test_gpu_parity.py tests/test_large_parity.py -m gpu -x -q 2>&1 | tail -1
run() { env $1 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$1', round(d['ms_per_step'],4), round(d['roofline']['p2p_ms'],4), d['launches_per_step'])" 2>/dev/null || tail -1 gpurun_out/ab.err; }
for r in 1 2; do run X=1; run VFMM_SYM_FUSED_SUM=1; done
