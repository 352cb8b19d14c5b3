# 1-GPU A/B of K1 builds (vectors per thread, min CTAs per SM), alternating (development script)
O=gpurun_out/r2ac
mkdir -p $O
L=paper_2407_07852_b200/libdiloco_cuda.so
cp $L /tmp/lib_product.so
for rep in 1 2 3; do
  for v in product mb8 u2 u2mb4; do
    if [ $v = product ]; then cp /tmp/lib_product.so $L; else cp paper_2407_07852_b200/variants/$v/libdiloco_cuda.so $L; fi
    echo "{\"variant\": \"$v\", \"r\": $(timeout 120 python tools/k1_probe.py)}" >> $O/k1_ab.jsonl 2>> $O/k1_ab.err
  done
done
cp /tmp/lib_product.so $L
echo done
