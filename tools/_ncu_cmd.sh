set -x
ncu --set full --import-source on --clock-control none -k replay_kernel -c 1 -o gpurun_out/pair27_full python tools/ncu_target.py C2 27 28 > gpurun_out/ncu_pair27.log 2>&1
ncu -i gpurun_out/pair27_full.ncu-rep --page source --csv --print-source sass > gpurun_out/pair27_sass.csv 2>/dev/null
ncu -i gpurun_out/pair27_full.ncu-rep --page source --csv --print-source cuda > gpurun_out/pair27_src.csv 2>/dev/null
ls -la gpurun_out
