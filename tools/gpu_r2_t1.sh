set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
free -g | head -2; nproc
timeout 1500 python -m pytest tests -q -m gpu -x -k "graph_replay or neural_7b or stochastic" -s 2>&1 | tail -40 > gpurun_out/r2_t1.log
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -15 >> gpurun_out/r2_t1.log
