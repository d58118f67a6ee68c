( for c in 2 3; do python tools/m2l_probe.py $c; done
  VFMM_M2L_CW=3 python tools/m2l_probe.py 2
  VFMM_M2L_CW=1 python tools/m2l_probe.py 3
  VFMM_M2L_CW=2 python tools/m2l_probe.py 3
 ) > gpurun_out/m2l_probe.log 2>&1
cat gpurun_out/m2l_probe.log
