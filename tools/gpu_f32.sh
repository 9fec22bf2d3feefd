mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_f32_gpu.py -q -x 2>&1 | tail -15
