timeout 400 python -m pytest tests/test_gpu_stream_dit.py tests/test_gpu_pipeline.py tests/test_gpu_dit_forward.py tests/test_gpu_dit_xl.py tests/test_gpu_bench_shape.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -1
VARIANTS="" bash tools/ncu_final_ab.sh 2>&1 | grep duration
