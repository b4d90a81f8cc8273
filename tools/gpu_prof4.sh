mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grp_reduce_pdl|k_grp_fwd_pdl" -s 300 -c 2 -o gpurun_out/p4_tb python bench.py --config terabyte --no-cpu --no-e2e --records 8000000 --steps 1 --warmup 1 > gpurun_out/p4_1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gs_units|k_gs_links|k_gs_records" -c 3 -o gpurun_out/p4_group python bench.py --no-cpu --no-e2e --records 4000000 --steps 1 --warmup 1 > gpurun_out/p4_2.log 2>&1
du -sh gpurun_out/p4*
