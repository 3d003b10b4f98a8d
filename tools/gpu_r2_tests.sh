#!/bin/bash
# full GPU suite + smoke (round-2 final state)
mkdir -p gpurun_out/r02
nvidia-smi -L > gpurun_out/r02/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r02/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02/smoke.log
tail -4 gpurun_out/r02/pytest_gpu.log; cat gpurun_out/r02/smoke.log
