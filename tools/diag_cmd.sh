SILENZIO_LIB=tools/libsilenzio_pf.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pbs or blind" > gpurun_out/diag32.txt 2>&1
for L in paper_2504_17785_b200/libsilenzio.so tools/libsilenzio_pf.so tools/libsilenzio_pfd.so; do
  SILENZIO_LIB=$L timeout 300 python tools/time_br.py --batch 8880 --reps 3 >> gpurun_out/diag32.txt 2>&1
done
