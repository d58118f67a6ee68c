# ncu --set full (source-level) of the kernels matching a regex on one BASELINE config:
#   bash tools/ncu_kernel.sh <config> <regex> <out-name> [count]
cfg=$1; rx=$2; out=$3; cnt=${4:-4}
python tools/profile_graph.py $cfg 1 > gpurun_out/pg_$out.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$rx" -c $cnt -o gpurun_out/$out python tools/profile_graph.py $cfg 1 > gpurun_out/ncu_$out.log 2>&1
tail -2 gpurun_out/ncu_$out.log
