#!/bin/bash
# GEMM epilogue A/B (TLT_GEMM_EPI_ROUND 2 vs 1): GEMM + top-k tests, timings, engine parity subset, bench
mkdir -p gpurun_out
P=${1:-c2}
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_topk.py -q -x -p no:cacheprovider > gpurun_out/${P}_gemm_tests.log 2>&1; tail -5 gpurun_out/${P}_gemm_tests.log
shapes="272:3584:37888:3 528:3584:37888:3 272:18944:3584:2 528:18944:3584:2 528:3584:4608:0 528:3584:3584:2 496:3584:152064:0 17:3584:37888:3 17:18944:3584:2"
for v in 0 1 8; do for e in 2 1; do
  echo "== variant $v round $e"
  TLT_GEMM_FORCE_VARIANT=$v TLT_GEMM_EPI_ROUND=$e timeout 120 python tools/time_gemms.py $shapes 2>&1 | grep -v Warn
done; done > gpurun_out/${P}_epi_ab.txt
timeout 1500 python -m pytest tests/test_gpu_parity_tiny.py tests/test_gpu_neural_7b.py tests/test_gpu_parity_graphs.py -q -x -p no:cacheprovider > gpurun_out/${P}_parity.log 2>&1; tail -5 gpurun_out/${P}_parity.log
timeout 1500 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
