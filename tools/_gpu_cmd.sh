O=gpurun_out
timeout 120 python tools/trace_gemm.py 2>&1 | grep -E "event|wait"
