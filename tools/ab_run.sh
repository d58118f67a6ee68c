for v in "X=1" "VFMM_P2P_SPLIT=1" "VFMM_P2P_SPLIT=1 VFMM_P2P_SYM_K=2" "VFMM_P2P_SPLIT=1 VFMM_P2P_SYM_K=3"; do
  echo "$v: $(env $v python tools/shard_probe.py 2 8 2>&1 | tail -1 | cut -c1-120)"
done
for v in "X=1" "VFMM_P2P_SYM_K=2" "VFMM_P2P_SPLIT=1 VFMM_P2P_SYM_K=2"; do
  echo "$v: $(env $v python tools/phase_probe.py 1 2>&1 | tail -1)"
done
