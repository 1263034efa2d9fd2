O=gpurun_out/r2g; mkdir -p $O; rm -f $O/*
for ns in 2 3 4 2 3 4; do SPARSEB200_STREAM_NS=$ns timeout 600 python tools/sweep_configs.py --skip-cpu --only 1,2 > $O/s$ns.json 2>/dev/null; python -c "
import json
d=json.load(open('$O/s$ns.json'))
print('ns=$ns c1', round(d['config1_poisson2d_1000_csr_f64']['us'],2), {k:round(v['csr']['us'],1) for k,v in d['config2_poisson128_formats'].items()})" >> $O/ns.log; done
cat $O/ns.log
