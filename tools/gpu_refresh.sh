mkdir -p gpurun_out/refresh
for c in kaggle terabyte alibaba; do
timeout 900 python bench.py --mixed --config $c > gpurun_out/refresh/mixed_$c.log 2>&1
done
for c in kaggle terabyte; do
timeout 900 python bench.py --exchange --config $c --no-cpu --no-e2e > gpurun_out/refresh/exchange_$c.log 2>&1
done
timeout 1500 python bench.py --sweep > gpurun_out/refresh/sweep.log 2>&1
