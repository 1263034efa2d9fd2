O=gpurun_out/r2f; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_formats.py tests/test_gpu_solvers.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
