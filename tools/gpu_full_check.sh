#!/bin/bash
# full GPU pass: every -m gpu test, smoke, the default bench line
mkdir -p gpurun_out
P=${1:-full}
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${P}_tests_full.log 2>&1; tail -15 gpurun_out/${P}_tests_full.log > gpurun_out/${P}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
