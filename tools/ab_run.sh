run() { env $1 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$1', round(d['ms_per_step'],4), d['launches_per_step'])" || tail -3 gpurun_out/ab.err; }
run X=1
run VFMM_PRIO_M2L=1
run "VFMM_PRIO_M2L=1 VFMM_NEAR_AFTER=none"
run X=1
