O=gpurun_out/r2c; mkdir -p $O; rm -f $O/*
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_persistent -s 1 -c 1 -o $O/cg2 python tools/cg_ab.py 128 > $O/ncu.log 2>&1
SPARSEB200_CG_PROFILE=1 timeout 120 python tools/cg_ab.py 128 > $O/phases.log 2>&1
tail -5 $O/phases.log
