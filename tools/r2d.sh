O=gpurun_out/r2d; mkdir -p $O; rm -f $O/ab.log
timeout 600 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2 3; do for d in 2 0 1; do for p in 128 64; do SPARSEB200_CG_DYN=$d timeout 120 python tools/cg_ab.py $p 2>&1 | head -1 | sed "s/^/dyn=$d /" >> $O/ab.log; done; done; done
tail -3 $O/pytest.log; cat $O/ab.log
