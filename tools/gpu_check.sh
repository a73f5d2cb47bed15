# GPU iteration loop: parity tests, then per-pair timing of the C2 search.
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
python tools/pair_profile.py ${1:-C2} > gpurun_out/pair_profile.json 2>&1
python tools/profile_summary.py gpurun_out/pair_profile.json
