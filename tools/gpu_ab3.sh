mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
for i in 1 2; do
for v in libfae libfae_tiny8; do
FAE_VERBOSE=1 FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --no-cpu --no-e2e --records 24000000 --steps 4 --warmup 3 > gpurun_out/ab3_${v}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab3_${v}_$i.log >> gpurun_out/ab3_summary.txt; echo "$v $i" >> gpurun_out/ab3_summary.txt
grep "avg after\|last reduce" gpurun_out/ab3_${v}_$i.log | tail -2 >> gpurun_out/ab3_summary.txt
done; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_grp_" -s 4000 -c 400 --csv --log-file gpurun_out/ab3_launches_tb16m.csv python bench.py --no-cpu --no-e2e --records 16000000 --steps 1 --warmup 1 > gpurun_out/ab3_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grp_reduce_pdl|k_grp_fwd_pdl" -s 300 -c 2 -o gpurun_out/ab3_full_tb python bench.py --no-cpu --no-e2e --records 16000000 --steps 1 --warmup 1 > gpurun_out/ab3_ncu_full.log 2>&1
du -sh gpurun_out/ab3*
