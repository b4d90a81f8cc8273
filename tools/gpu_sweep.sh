mkdir -p gpurun_out
for B in 2048 8192 32768 65536; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 2 --records 20000000 --batch $B > gpurun_out/sw_k_$B.log 2>&1
done
for B in 4096 16384; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 2 --records 20000000 --batch $B --config terabyte > gpurun_out/sw_tb_$B.log 2>&1
done
