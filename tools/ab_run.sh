for rep in 1 2; do
for lib in default build/s2/libvfmm.so build/s2r2/libvfmm.so; do
  if [ "$lib" = default ]; then e=""; else e="VFMM_LIB=$lib"; fi
  echo "$lib: $(env $e X=1 python tools/phase_probe.py 2 2>&1 | tail -1 | cut -c1-150)"
done
done
echo "c1 default $(python tools/phase_probe.py 1 | tail -1)"
echo "c1 s2 $(VFMM_LIB=build/s2/libvfmm.so python tools/phase_probe.py 1 | tail -1)"
