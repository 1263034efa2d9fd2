O=gpurun_out/r2d; mkdir -p $O; rm -f $O/ab.log
for p in 160 192 256 320; do for pm in 0 100000; do
 if [ $pm = 0 ]; then SPARSEB200_CG_FUSED=1 timeout 300 python tools/cg_ab.py $p 2>&1 | head -1 | sed "s/^/graph /" >> $O/ab.log;
 else SPARSEB200_CG_PMAX_MB=$pm timeout 300 python tools/cg_ab.py $p 2>&1 | head -1 | sed "s/^/persistent /" >> $O/ab.log; fi
done; done
cat $O/ab.log
