# SMPC iteration loop on the GPU box: planner parity tests, M sweep, phase trace.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_planner.py tests/test_gpu_production.py -x -q > gpurun_out/pt_planner.log 2>&1; echo "rc=$?" >> gpurun_out/pt_planner.log
timeout 300 python tools/m_sweep.py --ms 4,4096,8192 > gpurun_out/m_sweep.json 2>&1
timeout 300 python tools/smpc_trace.py --flush > gpurun_out/trace_flush.json 2>/dev/null
timeout 300 python tools/smpc_trace.py --flush --samples 4 > gpurun_out/trace4_flush.json 2>/dev/null
