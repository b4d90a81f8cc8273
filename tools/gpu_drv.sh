mkdir -p gpurun_out
s=$(date +%s); timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_bench.log 2>&1; echo "bench wall $(( $(date +%s) - s )) s" > gpurun_out/drv_time.log
s=$(date +%s); timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_ref.log 2>&1; echo "ref wall $(( $(date +%s) - s )) s" >> gpurun_out/drv_time.log
