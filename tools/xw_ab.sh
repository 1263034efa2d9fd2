#!/bin/bash
# A/B of the persistent-CG x update in the barrier waits (SPARSEB200_CG_XW) on one box
O=gpurun_out/xw; mkdir -p $O; T=${1:-ab}
for rep in 1 2 3; do
  for xw in ${XWS:-0 1 2}; do SPARSEB200_CG_XW=$xw timeout 120 python tools/cg_ab.py 128 2>&1 | grep per-iter | sed "s/^/xw=$xw /"; done
done | tee $O/$T.txt
for xw in ${XWS:-0 1 2}; do SPARSEB200_CG_XW=$xw SPARSEB200_CG_PROFILE=1 timeout 120 python tools/cg_ab.py 128 2>&1 | grep "persistent CG" | tail -1 | sed "s/^/xw=$xw /"; done | tee -a $O/$T.txt
for p in 64 96 160; do for xw in ${XWS:-0 1 2}; do SPARSEB200_CG_XW=$xw timeout 120 python tools/cg_ab.py $p 2>&1 | grep per-iter | sed "s/^/xw=$xw /"; done; done | tee -a $O/$T.txt
for xw in ${XWS:-1 2}; do SPARSEB200_CG_XW=$xw timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "cg or Cg or solver or bench or frontend" 2>&1 | tail -1 | sed "s/^/xw=$xw /"; done | tee -a $O/$T.txt
