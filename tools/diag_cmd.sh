python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke3.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all2.log 2>&1; echo rc=$? >> gpurun_out/gpu_all2.log
