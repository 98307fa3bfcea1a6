timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gadgets.py -x -q > gpurun_out/diag40.txt 2>&1
python -c "
from paper_2504_17785_b200 import silenzio
from synth import get_params
P=get_params('A'); print('launches 131072:', silenzio.pbs_launch_count(P, 131072), 'for 1:', silenzio.pbs_launch_count(P, 1))" >> gpurun_out/diag40.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench11.json 2> gpurun_out/bench11.err
