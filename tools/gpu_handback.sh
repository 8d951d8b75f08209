#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_handback.py tests/test_ngram.py -m gpu -q > gpurun_out/pytest_hb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hb.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_hb.log
