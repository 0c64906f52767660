./build/k2_cluster_probe 2 2>&1 | grep -v "^  sm"
timeout 900 python -m pytest tests/test_gpu_long.py tests/test_gpu_shapes.py tests/test_gpu_parity.py -q -x 2>&1 | tail -5
python tools/stream_flush_ab.py 1; python tools/stream_flush_ab.py 0
bash tools/gpu_sanitize.sh
