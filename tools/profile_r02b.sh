# Round-2 (second session) evidence run: default bench line, reference arm,
# ncu launch list of graph replays and ncu --set full of one replay (config 2),
# the near-field kernel of config 3, and the emulated shard probe.
set -x
python bench.py > gpurun_out/r02b_bench_config2.json 2> gpurun_out/r02b_bench_config2.err
python bench.py --impl reference > gpurun_out/r02b_bench_reference_arm.json 2> gpurun_out/r02b_bench_reference_arm.err
python tools/profile_graph.py 2 3 > gpurun_out/pg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_config2_graph.csv python tools/profile_graph.py 2 3 > gpurun_out/ncu_l2.log 2>&1
ncu --set full --clock-control none --import-source on --launch-skip 21 -c 12 -o gpurun_out/r02b_graph_config2 python tools/profile_graph.py 2 2 > gpurun_out/ncu_f2.log 2>&1
python tools/profile_graph.py 3 1 > gpurun_out/pg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_p2p_sym|k_m2l_tile" --launch-skip 0 -c 2 -o gpurun_out/r02b_config3 python tools/profile_graph.py 3 1 > gpurun_out/ncu_f3.log 2>&1
python tools/shard_probe.py 2 1 2 4 8 > gpurun_out/r02b_shard_probe.txt 2>&1
python tools/shard_probe.py 3 8 >> gpurun_out/r02b_shard_probe.txt 2>&1
ls -la gpurun_out/
