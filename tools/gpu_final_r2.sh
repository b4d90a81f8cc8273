mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/f_bench_tb.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.log 2>&1
