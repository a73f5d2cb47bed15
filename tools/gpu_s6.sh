mkdir -p gpurun_out/san
for t in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 200 python tools/sanitize.py > gpurun_out/san/${t}.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/san/rc.txt
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_s6.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:replay_kernel -c 1 -o gpurun_out/c2_s6 python tools/ncu_target.py C2 > gpurun_out/ncu_c2_s6.log 2>&1
ncu -i gpurun_out/c2_s6.ncu-rep --page raw --csv > gpurun_out/c2_s6_raw.csv 2>/dev/null
ncu -i gpurun_out/c2_s6.ncu-rep --page source --csv > gpurun_out/c2_s6_source.csv 2>/dev/null
rm -f gpurun_out/c2_s6.ncu-rep
echo done
