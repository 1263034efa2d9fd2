O=gpurun_out/r2g; mkdir -p $O; rm -f $O/*
for r in 0 1 0 1; do
SPARSEB200_SOLVER_R128=$r timeout 900 python tools/sweep_configs.py --skip-cpu --only 4 > $O/s4_$r.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/s4_$r.json'))['config4_convdiff256_f64']; print('r128=$r', {k:round(v['ms_per_iteration'],4) for k,v in d.items()})" >> $O/r.log
SPARSEB200_SOLVER_R128=$r SPARSEB200_CG_FUSED=1 timeout 300 python tools/cg_ab.py 256 2>&1 | head -1 | sed "s/^/r128=$r cg256 /" >> $O/r.log
done
cat $O/r.log
