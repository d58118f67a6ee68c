./tools/ubench/ring4 200
python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print('bench', d['value']/1e9, d['ms_per_step'], 'e2e', d['e2e']['value']/1e9, d['phases_ms'], d['roofline']['build'])"
python tools/phase_probe.py 2
python tools/phase_probe.py 1
VFMM_SORT=lsd python tools/phase_probe.py 2
