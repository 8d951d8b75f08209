#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ngram.py -m gpu -q > gpurun_out/pytest_ngram.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ngram.log
tail -30 gpurun_out/pytest_ngram.log
