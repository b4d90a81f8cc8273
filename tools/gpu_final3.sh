mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/h_bench_kaggle.log 2>&1
timeout 900 python bench.py --config terabyte --no-cpu > gpurun_out/h_bench_tb.log 2>&1
