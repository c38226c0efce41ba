nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt; nvidia-smi > gpurun_out/smi.txt 2>&1
python -c "import numpy, scipy; print(numpy.__version__, scipy.__version__)" >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
