timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k full_batch > gpurun_out/diag29.txt 2>&1
