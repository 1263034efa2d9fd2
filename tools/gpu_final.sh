#!/bin/bash
# Round-end evidence pass on one B200 (run under gpurun from the repo root):
#   GPU suite, smoke, bench (ours + reference arm), ncu launch list of the bench command,
#   ncu --set full of the persistent CG kernel and the stream SpMV, config sweep.
TAG=${1:-r2final}
O=gpurun_out/$TAG
mkdir -p $O; rm -f $O/*
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:cg_persistent -s 1 -c 1 -o $O/cg python tools/cg_ab.py 128 > $O/ncu_cg.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:csr_stream_kernel -s 3 -c 1 -o $O/spmv python tools/prof_cg.py 128 > $O/ncu_spmv.log 2>&1
[ -z "$SKIP_SWEEP" ] && timeout 1500 python tools/sweep_configs.py --skip-cpu > $O/sweep.json 2> $O/sweep.err
tail -2 $O/pytest_gpu.log; cat $O/smoke.log | tail -1; cut -c1-300 $O/bench.json
# post-process the --set full reports on the box (the .ncu-rep files exceed the 64 MiB copy-back)
for r in cg spmv; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page details > $O/${r}_details.txt 2>/dev/null
  python tools/ncu_table.py $O/$r.ncu-rep > $O/${r}_table.txt 2>/dev/null
done
python tools/traffic_json.py $O/cg.ncu-rep cg_persistent $O/cg_traffic.json 320 384696324 > /dev/null 2>&1
python tools/traffic_json.py $O/spmv.ncu-rep csr_stream $O/spmv_traffic.json 1 216924164 > /dev/null 2>&1
rm -f $O/cg.ncu-rep; mv $O/spmv.ncu-rep $O/spmv_keep.ncu-rep
du -sh $O
