#!/bin/bash
# A/B: BR-only time at 131072 and per-launch DRAM bytes (ncu) for the default library and variants
mkdir -p gpurun_out
for v in default rs1 rs2; do
  if [ $v = default ]; then L=$PWD/paper_2504_17785_b200/libsilenzio.so; else L=$PWD/tools/libsilenzio_$v.so; fi
  SILENZIO_LIB=$L timeout 200 python tools/time_br.py --batch 131072 --reps 2
  SILENZIO_LIB=$L timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
     -k regex:blind_rotate_warp -c 1 --csv python tools/time_br.py --batch 131072 --reps 1 2>/dev/null | grep -E "dram__bytes|lts__t_bytes" | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
