# 1-GPU: smoke, the whole GPU suite, bench and its ncu launch list at HEAD (development script)
O=gpurun_out/r2f
mkdir -p $O
nproc > $O/nproc.txt; free -g >> $O/nproc.txt; nvidia-smi -L >> $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > $O/pytest_gpu.log 2>&1
timeout 300 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/ref.json 2> $O/ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
echo done
