timeout 900 python -m pytest tests/test_gpu_setc.py tests/test_gpu_setb.py -x -q > gpurun_out/diag31.txt 2>&1
for L in paper_2504_17785_b200/libsilenzio.so tools/libsilenzio_ctm0.so; do
  SILENZIO_LIB=$L timeout 600 python tools/time_setb.py --params C --batch 592 >> gpurun_out/diag31.txt 2>&1
done
SILENZIO_LIB=paper_2504_17785_b200/libsilenzio.so timeout 600 python tools/time_setb.py --params B --batch 296 >> gpurun_out/diag31.txt 2>&1
