python -m pytest tests/test_gpu_parity.py tests/test_large_parity.py tests/test_distributed.py -m gpu -x -q 2>&1 | tail -2
for c in 1 2 3; do python tools/m2l_probe.py $c; done
python tools/shard_probe.py 2 8 2>&1 | tail -1
VFMM_M2L_TG=2 python tools/shard_probe.py 2 8 2>&1 | tail -1
python bench.py --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "import json; d=json.load(open('gpurun_out/b.json')); print(d['ms_per_step'], d['roofline']['m2l'], d['roofline']['build'], d['roofline']['step'], d['e2e']['value']/1e9)"
