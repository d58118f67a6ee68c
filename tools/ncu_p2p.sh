# ncu --set full of the symmetric near-field kernel on config 2 (source-level stall sampling)
set -x
python tools/profile_graph.py 2 1 > gpurun_out/pg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_p2p_sym" -c 1 -o gpurun_out/p2p_cur python tools/profile_graph.py 2 1 > gpurun_out/ncu_p2p.log 2>&1
tail -3 gpurun_out/ncu_p2p.log
