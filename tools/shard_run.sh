python -m pytest tests/test_distributed.py tests/test_gpu_api.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
PHASES=1 python tools/shard_probe.py 2 1 8 2>&1 | tail -8
for c in 1 2 3; do python tools/m2l_probe.py $c; done
VFMM_M2L_TG=3 python tools/m2l_probe.py 2
VFMM_M2L_TG=3 python tools/m2l_probe.py 1
