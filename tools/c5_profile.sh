# Throughput-config profile: whole-kernel stalls and per-SASS-address
# execution counts of the replay kernel over ~1.1 waves of C5 pairs.
python tools/ncu_target.py C5 0 3400 1 > gpurun_out/c5_plain.log 2>&1; tail -1 gpurun_out/c5_plain.log
ncu --set full --import-source on --clock-control none -k regex:replay_kernel -c 1 -o gpurun_out/c5_full python tools/ncu_target.py C5 0 3400 1 > gpurun_out/ncu_c5.log 2>&1
ncu -i gpurun_out/c5_full.ncu-rep --page raw --csv > gpurun_out/c5_full_raw.csv 2>/dev/null
ncu -i gpurun_out/c5_full.ncu-rep --page source --csv --print-source sass > gpurun_out/c5_sass.csv 2>/dev/null
ls -la gpurun_out/c5_*
