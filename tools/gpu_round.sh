#!/bin/bash
# One gpurun call: GPU parity tests, smoke, 1-GPU bench, launch list.
#   gpurun --timeout 1800 -- 'bash tools/gpu_round.sh'
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ "${LAUNCHES:-1}" = 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 1 --sd 2 --strategy 6,8,16 > gpurun_out/launches.log 2>&1
echo "ncu rc=$?" >> gpurun_out/launches.log
fi
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
