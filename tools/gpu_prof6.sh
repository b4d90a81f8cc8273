mkdir -p gpurun_out
timeout 300 python bench.py --train --config terabyte --records 4000000 --no-cpu --no-e2e > gpurun_out/p6_train.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_|gemm|cutlass|nvjet|sm100|Kernel" -s 3000 -c 600 --csv --log-file gpurun_out/p6_launches_train_tb4m.csv python bench.py --train --config terabyte --records 4000000 --no-cpu --no-e2e > gpurun_out/p6_ncu.log 2>&1
ls -la gpurun_out/p6*
