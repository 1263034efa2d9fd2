O=gpurun_out/r2g; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -p no:cacheprovider -k split > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
