# 1-GPU: ncu --set full of the fused boundary kernels (pingpong, 6 CTAs per SM) at 1.1B (development script)
O=gpurun_out/r2aq
mkdir -p $O
python tools/boundary_probe.py > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:boundary_solo_kernel -c 2 -o $O/prof_boundary python tools/boundary_probe.py > $O/ncu.log 2>&1
echo done
