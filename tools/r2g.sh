O=gpurun_out/r2g; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -p no:cacheprovider -k "tile or powerlaw or golden" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/sweep_configs.py --skip-cpu --only 3 > $O/sweep.json 2> $O/sweep.err
tail -2 $O/pytest.log
