# C3 headline profile set: DRAM bytes per launch of the full C3 search (the
# bench's roofline.traffic), ncu --set full of the C3s search (same pairs and
# concurrency, 10k-session replicas), candidate attainment spread at the rate.
set -x
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:replay_kernel -c 1 --csv --log-file gpurun_out/traffic_c3.csv python tools/ncu_target.py C3 > gpurun_out/traffic_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:replay_kernel -c 1 -o gpurun_out/c3s_full \
    python tools/ncu_target.py C3s > gpurun_out/ncu_c3s.log 2>&1
ncu -i gpurun_out/c3s_full.ncu-rep --page raw --csv > gpurun_out/c3s_full_raw.csv 2>/dev/null
ncu -i gpurun_out/c3s_full.ncu-rep --page source --csv > gpurun_out/c3s_full_source.csv 2>/dev/null
python tools/c3_rates.py 2.0 > gpurun_out/c3_rates.log 2>&1
ls -la gpurun_out
