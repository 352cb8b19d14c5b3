# 2/4-GPU A/B: exchange stores / loads with default caching (variants/l2) vs streaming hints (product), alternating builds (development script)
# builds the variant first: make -C paper_2407_07852_b200/csrc EXTRA=-DDLC_EXCHANGE_L2 BUILD=/tmp/build_l2 OUT=$PWD/paper_2407_07852_b200/variants/l2/libdiloco_cuda.so
O=gpurun_out/r2v
mkdir -p $O
L=paper_2407_07852_b200/libdiloco_cuda.so
cp $L /tmp/lib_product.so
for n in 4 2; do
  for rep in 1 2 3; do
    for v in product l2; do
      if [ $v = product ]; then cp /tmp/lib_product.so $L; else cp paper_2407_07852_b200/variants/l2/libdiloco_cuda.so $L; fi
      echo "# $v rep $rep" >> $O/ab_${n}gpu.log
      CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n tools/sweep_p2p.py --no-ordered --steps 10 --repeat 2 >> $O/ab_${n}gpu.log 2>> $O/ab_${n}gpu.err
    done
  done
done
cp /tmp/lib_product.so $L
echo done
