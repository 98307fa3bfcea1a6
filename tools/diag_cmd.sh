timeout 600 python tools/time_setb.py --params B --batch 148 >> gpurun_out/diag35.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_setb.py -x -q >> gpurun_out/diag35.txt 2>&1
