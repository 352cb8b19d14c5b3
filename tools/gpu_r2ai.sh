# 1-GPU A/B of the INPLACE fused boundary's min CTAs per SM (development script)
O=gpurun_out/r2ai
mkdir -p $O
L=paper_2407_07852_b200/libdiloco_cuda.so
cp $L /tmp/lib_product.so
for rep in 1 2; do
  for v in product imb6; do
    if [ $v = product ]; then cp /tmp/lib_product.so $L; else cp paper_2407_07852_b200/variants/$v/libdiloco_cuda.so $L; fi
    timeout 300 python bench.py --inner-mode inplace --no-e2e --no-cpu-baseline --no-wire --no-training > $O/bench_${v}_${rep}.json 2> $O/bench_${v}_${rep}.err
  done
done
cp /tmp/lib_product.so $L
echo done
