set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
for c in config0 overlap config1 generic bigleaf graph direct at shard; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_cases.py $c > gpurun_out/san_racecheck_$c.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck_$c.log
done
tail -n 3 gpurun_out/san_*.log
