# evidence: launch list + ncu --set full of the dominant train kernels (Kaggle fused, Terabyte 2-kernel)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q_launches_kaggle10m.csv python bench.py --no-cpu --no-e2e --records 10000000 --steps 1 --warmup 1 > gpurun_out/q_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grp_fused_pdl" -s 3000 -c 3 -o gpurun_out/q_full_fused python bench.py --no-cpu --no-e2e --records 10000000 --steps 1 --warmup 1 > gpurun_out/q_ncu_full1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grp_reduce_pdl|k_grp_fwd_pdl" -s 2000 -c 4 -o gpurun_out/q_full_tb python bench.py --config terabyte --no-cpu --no-e2e --records 8000000 --steps 1 --warmup 1 > gpurun_out/q_ncu_full2.log 2>&1
