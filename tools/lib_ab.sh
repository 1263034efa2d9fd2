#!/bin/bash
# same-box A/B of two builds of the library (SPARSEB200_LIB): CG 128^3 per iteration and the
# 128^3 format sweep + config #1 (tools/sweep_configs.py --only 1,2)
O=gpurun_out/libab; mkdir -p $O
for rep in 1 2 3; do
  for L in "$@"; do SPARSEB200_LIB=$L timeout 120 python tools/cg_ab.py 128 2>&1 | grep per-iter | sed "s|^|$L |"; done
done | tee $O/cg.txt
for L in "$@"; do
  SPARSEB200_LIB=$L timeout 600 python tools/sweep_configs.py --skip-cpu --only 1,2 > $O/sweep_$(basename $L).json 2>/dev/null
  python - $O/sweep_$(basename $L).json $L <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[2], "cfg1", round(d["config1_poisson2d_1000_csr_f64"]["us"], 2),
      {dt: {k: round(v["us"], 1) for k, v in r.items() if k != "coo_segmented"} for dt, r in d["config2_poisson128_formats"].items()})
PY
done | tee -a $O/cg.txt
