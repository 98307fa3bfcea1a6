timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "keyswitch or full_batch or config0" > gpurun_out/diag36.txt 2>&1
timeout 600 python tools/kst_bench.py >> gpurun_out/diag36.txt 2>&1
