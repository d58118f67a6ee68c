set -x
python tools/profile_graph.py 2 3 > gpurun_out/pg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_config2.csv python tools/profile_graph.py 2 3 > gpurun_out/ncu_l2.log 2>&1
python tools/profile_graph.py 2 1 > gpurun_out/pg2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_p2p_sym|k_m2l_tile|k_l2l_fused|k_leaf_pack|k_bin_count|k_bin_scatter|k_near_sum|k_p2m_grp|k_m2m_subtree|k_zero_regions|k_scan_one|k_counts_tasks" -c 14 -o gpurun_out/r02_full_config2 python tools/profile_graph.py 2 1 > gpurun_out/ncu_f2.log 2>&1
python tools/profile_graph.py 3 1 > gpurun_out/pg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_p2p_sym|k_m2l_tile" -c 2 -o gpurun_out/r02_full_config3 python tools/profile_graph.py 3 1 > gpurun_out/ncu_f3.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
