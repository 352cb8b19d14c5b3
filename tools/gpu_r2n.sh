# 1-GPU: ncu --set full of the fused single-worker boundary kernel; launch list of bench (development script)
O=gpurun_out/r2n
mkdir -p $O
python tools/boundary_probe.py > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:boundary_solo_kernel -c 2 -o $O/prof_boundary python tools/boundary_probe.py > $O/ncu.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-wire --no-e2e --no-training > $O/bench_plain.json 2> $O/bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-wire --no-e2e --no-training > $O/ncu_launch.log 2>&1
echo done
