mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/c1_smi.txt
bash tools/gpu_gemm_diag.sh "0 1 2 8" > gpurun_out/c1_gemm_diag.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/c1_tests_full.log 2>&1; tail -15 gpurun_out/c1_tests_full.log > gpurun_out/c1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
