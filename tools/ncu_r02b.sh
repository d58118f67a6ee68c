# Round-2 (session 2) captures of config 2 as the bench runs it (graph replay):
# the launch list, then ncu --set full of every kernel of one replay.
set -x
python tools/profile_graph.py 2 3 > gpurun_out/pg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_config2.csv python tools/profile_graph.py 2 3 > gpurun_out/ncu_l2.log 2>&1
ncu --set full --clock-control none --import-source on --launch-skip 12 -c 12 -o gpurun_out/r02b_full_config2 python tools/profile_graph.py 2 2 > gpurun_out/ncu_f2.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
