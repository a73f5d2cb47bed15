# Throughput-config tuning: shared-memory budget per slot x slots per SM.
# SWEEP="budget:per_sm budget:per_sm ..." (per_sm 0 = as many as fit)
for cfg in ${SWEEP:-12288:32 8192:20 10240:22}; do
  b=${cfg%%:*}; n=${cfg##*:}
  if [ "$n" = "0" ]; then unset PDSIM_SLOTS_PER_SM; else export PDSIM_SLOTS_PER_SM=$n; fi
  PDSIM_SMEM_BUDGET=$b python tools/ncu_target.py ${CFG:-C5} 0 -1 2 2>&1 | tail -1 | sed "s/^/${CFG:-C5} smem=$b per_sm=$n /"
done
