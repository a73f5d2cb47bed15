# Round-end measurement set: C2 bench + reference arm + launch list + ncu full
# (tools/round_profile.sh), then the C1 / C3 / C5-slice bench lines.
bash tools/round_profile.sh
python bench.py --config C1 --steps 5 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config C3 --steps 1 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -1 gpurun_out/bench_c1.json; tail -1 gpurun_out/bench_c3.json; tail -1 gpurun_out/bench_c5.json
