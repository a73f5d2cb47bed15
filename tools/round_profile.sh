# One GPU call: bench line, ncu launch list of one bench step, ncu --set full
# of the replay kernel over the whole C2 search (traffic + stall summary).
set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:replay_kernel -c 1 -o gpurun_out/c2_full python tools/ncu_target.py C2 > gpurun_out/ncu_c2.log 2>&1
ncu -i gpurun_out/c2_full.ncu-rep --page raw --csv > gpurun_out/c2_full_raw.csv 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -1 gpurun_out/bench.json; tail -1 gpurun_out/bench_ref.json
