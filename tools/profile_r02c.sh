# Round-2 (third session) evidence run: default bench line, ncu launch list of
# the bench command itself and of graph replays, ncu --set full of every kernel
# of one stream-launched evaluate (config 2), the probes behind DESIGN.md §5c,
# the emulated shard probe.
set -x
python bench.py > gpurun_out/r02c_bench_config2.json 2> gpurun_out/r02c_bench_config2.err
python tools/overlap_probe.py 2 > gpurun_out/r02c_overlap_probe.txt 2>&1
python tools/pipe_c_probe.py 64 > gpurun_out/r02c_pipe_c_probe.txt 2>&1
python tools/duplex_probe.py > gpurun_out/r02c_duplex_probe.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-depth 2 > gpurun_out/pre.json 2>gpurun_out/pre.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-depth 2 > gpurun_out/ncu_lb.log 2>&1
python tools/profile_graph.py 2 3 > gpurun_out/pg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches_config2_graph.csv python tools/profile_graph.py 2 3 > gpurun_out/ncu_l2.log 2>&1
ncu --set full --clock-control none --import-source on -c 20 -o gpurun_out/r02c_stream_config2 python tools/profile_graph.py 2 1 > gpurun_out/ncu_f2.log 2>&1
python tools/shard_probe.py 2 1 2 4 8 > gpurun_out/r02c_shard_probe.txt 2>&1
python tools/shard_probe.py 3 8 >> gpurun_out/r02c_shard_probe.txt 2>&1
for c in 0 1 3; do python tools/phase_probe.py $c >> gpurun_out/r02c_phase_probe.txt 2>&1; done
ls -la gpurun_out/
