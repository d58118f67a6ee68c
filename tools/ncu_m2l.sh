# ncu --set full of the tiled M2L kernel on configs 2 and 3 (one capture each)
python tools/m2l_probe.py 2 3 > gpurun_out/ncu_m2l_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_m2l_tile -s 1 -c 1 -o gpurun_out/m2l_tile_c2 python tools/m2l_probe.py 2 3 > gpurun_out/ncu_m2l_c2.log 2>&1
python tools/m2l_probe.py 3 3 > gpurun_out/ncu_m2l_plain3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_m2l_tile -s 1 -c 1 -o gpurun_out/m2l_tile_c3 python tools/m2l_probe.py 3 3 > gpurun_out/ncu_m2l_c3.log 2>&1
ls -la gpurun_out/
