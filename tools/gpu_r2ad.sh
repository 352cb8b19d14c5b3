# 1-GPU A/B of K1 builds through bench.py's inner_adamw and window boundary (development script)
O=gpurun_out/r2ad
mkdir -p $O
L=paper_2407_07852_b200/libdiloco_cuda.so
cp $L /tmp/lib_product.so
for rep in 1 2; do
  for v in product u2mb4 mb8; do
    if [ $v = product ]; then cp /tmp/lib_product.so $L; else cp paper_2407_07852_b200/variants/$v/libdiloco_cuda.so $L; fi
    timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-wire --no-training > $O/bench_${v}_${rep}.json 2> $O/bench_${v}_${rep}.err
    timeout 120 python tools/k1_probe.py > $O/probe_${v}_${rep}.json 2>> $O/probe.err
  done
done
cp /tmp/lib_product.so $L
echo done
