mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_grp_" -s 4000 -c 400 --csv --log-file gpurun_out/p5_launches_tb16m.csv python bench.py --no-cpu --no-e2e --records 16000000 --steps 1 --warmup 1 > gpurun_out/p5_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grp_reduce_pdl|k_grp_fwd_pdl" -s 300 -c 2 -o gpurun_out/p5_full_tb python bench.py --no-cpu --no-e2e --records 16000000 --steps 1 --warmup 1 > gpurun_out/p5_ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p5_launches_bench_tb80m.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 0 > gpurun_out/p5_ncu_bench.log 2>&1
ls -la gpurun_out/p5*
