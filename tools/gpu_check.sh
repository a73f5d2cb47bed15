# GPU iteration loop: parity tests, then per-pair timing of the C2 search.
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
python tools/pair_profile.py ${1:-C2} > gpurun_out/pair_profile.json 2>&1
python - <<'PY'
import json
d=json.load(open('gpurun_out/pair_profile.json'))
print("kernel_ms", d["kernel_ms"], "top", [(t["pair"], t["cycles"], t["events"]) for t in d["top"][:3]])
for k,v in d["phases"].items(): print(k, v["count"], round(v["cycles_per"]))
PY
