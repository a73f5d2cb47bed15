# Round-2 evidence set for the committed build: bench line (default config and
# secondaries), reference arm, ncu launch list of a bench run, ncu --set full
# of the C3s search (throughput build) and C3 DRAM traffic per launch.
set -x
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --secondary none --no-argmax-mode > gpurun_out/b_ncu.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:replay_kernel -c 1 --csv --log-file gpurun_out/traffic_c3_final.csv python tools/ncu_target.py C3 > gpurun_out/traffic_final.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:replay_kernel -c 1 -o gpurun_out/c3s_final \
    python tools/ncu_target.py C3s > gpurun_out/ncu_c3s_final.log 2>&1
ncu -i gpurun_out/c3s_final.ncu-rep --page raw --csv > gpurun_out/c3s_final_raw.csv 2>/dev/null
ncu -i gpurun_out/c3s_final.ncu-rep --page source --csv > gpurun_out/c3s_final_source.csv 2>/dev/null
rm -f gpurun_out/c3s_final.ncu-rep
ls -la gpurun_out
