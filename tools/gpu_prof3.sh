# evidence: launch list + ncu --set full of the dominant train kernel (Kaggle fused); keep gpurun_out < 64 MiB
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "unit_path or grouped" 2>&1 | tail -3 > gpurun_out/q_pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q_launches_kaggle4m.csv python bench.py --no-cpu --no-e2e --records 4000000 --steps 1 --warmup 1 > gpurun_out/q_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grp_fused_pdl" -s 1500 -c 2 -o gpurun_out/q_full_fused python bench.py --no-cpu --no-e2e --records 4000000 --steps 1 --warmup 1 > gpurun_out/q_ncu_full1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gs_units|k_classify_fixed" -c 2 -o gpurun_out/q_full_units python bench.py --no-cpu --no-e2e --records 4000000 --steps 1 --warmup 1 > gpurun_out/q_ncu_full2.log 2>&1
du -sh gpurun_out/*
