# A/B of the graph conditional nodes and near-field start (bench value, graph replay)
run() { env $1 python bench.py --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$1', round(d['ms_per_step'],4), d['launches_per_step'], round(d['e2e']['value']/1e9,3))"; }
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_distributed.py -m gpu -x -q 2>&1 | tail -2
run VFMM_GRAPH_COND=0
run X=1
run VFMM_GRAPH_COND=0
run X=1
