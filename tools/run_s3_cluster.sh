# Round 2, third session: the fused analysis as one thread-block cluster (GPA_FUSED_CLUSTER)
set -x
GPA_LIB_PATH=$PWD/build/libcl16a.so timeout 900 python -m pytest tests -m gpu -x -q -k "fused or parity or estimate or advice" > gpurun_out/gt_cl16.log 2>&1; echo EXIT $? >> gpurun_out/gt_cl16.log
for l in ft ftcl16; do GPA_FT_LIB=$PWD/build/lib$l.so timeout 300 python tools/fused_timing.py 2 >> gpurun_out/ft_cl.txt 2>&1; done
WL="rodinia" bash tools/bench_ab.sh build/libcl16a.so build/libcl8a.so build/libfa.so > gpurun_out/ab_cl.txt 2>&1
