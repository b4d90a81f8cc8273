mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g_bench_tb.log 2>&1
timeout 900 python bench.py --config kaggle --steps 20 --warmup 5 > gpurun_out/g_bench_kaggle.log 2>&1
timeout 900 python bench.py --config alibaba --steps 20 --warmup 5 --no-cpu > gpurun_out/g_bench_ali.log 2>&1
