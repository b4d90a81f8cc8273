mkdir -p gpurun_out
start=$(date +%s)
timeout 1500 python bench.py > gpurun_out/t_bench.log 2>&1
end=$(date +%s)
echo "bench wall seconds: $((end-start))" >> gpurun_out/t_bench.log
start=$(date +%s)
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/t_ref.log 2>&1
end=$(date +%s)
echo "reference wall seconds: $((end-start))" >> gpurun_out/t_ref.log
