#!/bin/bash
# Quick end-state check: GPU suite, smoke, bench line
O=gpurun_out/check; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log; cut -c1-200 $O/bench.json
