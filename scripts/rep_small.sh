for i in $(seq 1 15); do timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "small_image_path_limits" 2>&1 | tail -1; done
