O=gpurun_out/r2d; mkdir -p $O; rm -f $O/ab.log
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_spmv.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do
for cfg in "2 4 0" "1 3 0"; do set -- $cfg
for p in 128 64; do
SPARSEB200_CG_SYNC=$1 SPARSEB200_CG1_MB=$2 timeout 120 python tools/cg_ab.py $p 2>&1 | head -1 | sed "s/^/sync=$1 mb=$2 /" >> $O/ab.log
done; done; done
timeout 300 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err
tail -3 $O/pytest.log; cat $O/ab.log; cut -c1-1500 $O/bench.json
