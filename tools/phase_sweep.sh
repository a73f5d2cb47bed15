for cfg in 256:8 128:16 64:24 32:32; do
  t=${cfg%%:*}; n=${cfg##*:}
  PDSIM_PHASE_THREADS=$t PDSIM_PHASE_CTAS_PER_SM=$n python -c "
import sys,time; sys.path.insert(0,'.')
from paper_2602_14516_b200 import native, workloads
prof=workloads.model_profile('llama3-8b'); st=native.preset_stats('toolbench')
trs=[native.gen_trace(st, (1.0+0.5*(k%32))*d/8.0, 256, 1000+k) for k in range(1024) for d in (1,2,4,8)]
with native.Context(0) as ctx:
    ctx.phase_sims([t.view for t in trs[:64]], [1,2,4,8]*16, prof)
    t0=time.perf_counter(); r=ctx.phase_sims([t.view for t in trs], [1,2,4,8]*1024, prof); dt=time.perf_counter()-t0
print('threads=$t per_sm=$n', round(dt,3), 's', r[5][1].p95)
"
done
