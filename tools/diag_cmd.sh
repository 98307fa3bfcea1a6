timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/diag8.txt 2>&1
for v in "" nowarp; do
  if [ -z "$v" ]; then L=paper_2504_17785_b200/libsilenzio.so; else L=tools/libsilenzio_$v.so; fi
  SILENZIO_LIB=$L timeout 300 python tools/time_br.py --batch 8880 --reps 3 >> gpurun_out/diag8.txt 2>&1
done
