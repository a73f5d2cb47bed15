# A/B of library variants on the throughput and latency configs:
# bash tools/gpu_ab.sh "LIB LIB ..." [CONFIGS] [ROUNDS]
libs=$1; cfgs=${2:-"C2 C5 C3s"}; rounds=${3:-2}
for c in $cfgs; do python tools/ab.py $c $rounds $libs; done 2>&1 | tee gpurun_out/ab.log
