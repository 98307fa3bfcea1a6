timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gadgets.py -x -q > gpurun_out/diag34.txt 2>&1
SILENZIO_LIB=paper_2504_17785_b200/libsilenzio.so timeout 300 python tools/time_br.py --batch 8880 --reps 3 >> gpurun_out/diag34.txt 2>&1
