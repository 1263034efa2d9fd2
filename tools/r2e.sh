O=gpurun_out/r2e; mkdir -p $O; rm -f $O/*
timeout 900 ncu --set full --clock-control none -k regex:"ell_kernel|sellp|csr_stream|csr_tile" -c 40 -o $O/formats python tools/prof_formats.py > $O/formats.log 2>&1
SPARSEB200_GRAPH=0 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/krylov.csv python tools/prof_krylov.py 256 512 > $O/krylov.log 2>&1
timeout 1200 python tools/sweep_configs.py --skip-cpu > $O/sweep.json 2> $O/sweep.err
ls -la $O; tail -3 $O/formats.log $O/krylov.log
