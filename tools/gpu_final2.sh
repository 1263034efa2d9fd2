#!/bin/bash
# Final-session evidence pass: GPU suite, smoke, bench (ours + reference arm), ncu launch
# list of the bench command, ncu --set full of the persistent CG kernel and of the 128^3
# format kernels (ELL / SELL-P / CSR stream, fp64 + fp32), full config sweep.
O=gpurun_out/r2fin; mkdir -p $O; rm -f $O/*
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"ell_kernel|sellp_block|csr_stream_kernel" -s 3 -c 40 -o $O/formats python tools/prof_formats.py > $O/ncu_formats.log 2>&1
python tools/ncu_table.py $O/formats.ncu-rep > $O/formats_table.txt 2>/dev/null; rm -f $O/formats.ncu-rep
timeout 1500 python tools/sweep_configs.py --skip-cpu > $O/sweep.json 2> $O/sweep.err
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log; cut -c1-300 $O/bench.json
du -sh $O
