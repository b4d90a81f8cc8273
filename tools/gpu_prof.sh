# round-1 evidence pass: GPU tests, full bench, launch list, ncu --set full of the top kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/p_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/p_bench_kaggle.log 2>&1
timeout 600 python bench.py --config terabyte --no-cpu --no-e2e > gpurun_out/p_bench_tb.log 2>&1
timeout 600 python bench.py --config alibaba --no-cpu --no-e2e > gpurun_out/p_bench_ali.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p_launches_kaggle10m.csv python bench.py --no-cpu --no-e2e --records 10000000 --steps 1 --warmup 1 > gpurun_out/p_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grp_reduce_pdl|k_grp_fwd_pdl" -s 2000 -c 4 -o gpurun_out/p_full_train python bench.py --no-cpu --no-e2e --records 10000000 --steps 1 --warmup 1 > gpurun_out/p_ncu_full1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gs_pass|k_gs_init|k_classify" -c 4 -o gpurun_out/p_full_group python bench.py --no-cpu --no-e2e --records 10000000 --steps 1 --warmup 1 > gpurun_out/p_ncu_full2.log 2>&1
