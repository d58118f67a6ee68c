python tools/shard_probe.py 2 8 2>&1 | tail -1
VFMM_GRAPH_COND=0 python tools/shard_probe.py 2 8 2>&1 | tail -1
python tools/phase_probe.py 1
