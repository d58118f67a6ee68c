# A/B of environment settings / library variants on the default bench (config 2):
#   bash tools/ab_run.sh "X=1" "VFMM_P2P_SYM_K=2" "VFMM_LIB=build/tabg/libvfmm.so" ...
run() { env $1 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$1', round(d['ms_per_step'],4), 'p2p', round(d['roofline']['p2p_ms'],4), 'build', round(d['roofline']['build']['ms'],4), 'down', round(d['phases_ms']['t_downward'],4), 'm2l', round(d['phases_ms']['t_m2l'],4), 'up', round(d['phases_ms']['t_upward'],4), d['launches_per_step']['graph_replay'])" 2>/dev/null || tail -1 gpurun_out/ab.err; }
for r in 1 2; do for a in "$@"; do run "$a"; done; done
