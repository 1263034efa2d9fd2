O=gpurun_out/r2c; mkdir -p $O; rm -f $O/*
timeout 600 ncu --set full --clock-control none --import-source on -k regex:persistent -s 1 -c 1 -o $O/cg1_staged python tools/cg_ab.py 128 > $O/ncu.log 2>&1
timeout 600 python -m pytest tests/test_gpu_solvers.py -x -q -p no:cacheprovider -k "persistent or cg" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
