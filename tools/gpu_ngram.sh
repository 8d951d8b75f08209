#!/bin/bash
# n-gram fallback drafter: GPU chain verify + rollout branch, then the full GPU suite.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ngram.py -m gpu -x -q > gpurun_out/pytest_ngram.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ngram.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
tail -30 gpurun_out/pytest_ngram.log
