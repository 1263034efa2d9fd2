mkdir -p gpurun_out/r2b
O=gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for p in 64 128; do for s in 1 2; do SPARSEB200_CG_SYNC=$s timeout 120 python tools/cg_ab.py $p >> $O/ab.log 2>&1; echo "sync=$s" >> $O/ab.log; done; done
for s in 1 2 1 2; do SPARSEB200_CG_SYNC=$s timeout 120 python tools/cg_ab.py 128 >> $O/ab.log 2>&1; echo "sync=$s" >> $O/ab.log; done
timeout 300 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err
tail -3 $O/pytest.log; cat $O/ab.log; cat $O/bench.json
