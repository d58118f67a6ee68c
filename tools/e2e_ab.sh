for r in 1 2; do for v in "VFMM_E2E_VARIANT=sync" "VFMM_E2E_VARIANT=copy" ; do
env $v python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --sharded --steps 3 --warmup 3 --e2e-steps 24 > gpurun_out/s.json 2> gpurun_out/s.err
python -c "import json; d=json.load(open('gpurun_out/s.json')); print('$v', round(d['e2e']['ms_per_step'],3), d['e2e']['h2d_bytes_per_step'])" || tail -3 gpurun_out/s.err
done; done
