O=gpurun_out/r2a
mkdir -p $O
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python -m pytest tests/test_world_gpu.py -x -q -rs > $O/world.log 2>&1
timeout 1500 python -m pytest tests/test_full_size.py -x -q -rs --durations=0 > $O/full.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rs --deselect tests/test_full_size.py --ignore=tests/test_full_size.py --ignore=tests/test_world_gpu.py > $O/rest.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
echo done
