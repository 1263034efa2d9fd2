O=gpurun_out/r2h; mkdir -p $O; rm -f $O/*
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_tile_kernel -s 1 -c 1 -o $O/tile python tools/prof_powerlaw.py csr > $O/ncu.log 2>&1
ncu -i $O/tile.ncu-rep --page source --csv --print-source sass > $O/tile_sass.csv 2>/dev/null
ncu -i $O/tile.ncu-rep --page raw --csv > $O/tile_raw.csv 2>/dev/null
rm -f $O/tile.ncu-rep; du -sh $O
