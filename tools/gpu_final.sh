mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/f_bench_kaggle.log 2>&1
timeout 600 python bench.py --config terabyte --no-cpu --no-e2e > gpurun_out/f_bench_tb.log 2>&1
timeout 600 python bench.py --config alibaba --no-cpu --no-e2e > gpurun_out/f_bench_ali.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_ref.log 2>&1
