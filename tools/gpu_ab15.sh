mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
for i in 1 2; do
for v in libfae libfae_o3 libfae_o1 libfae_o4; do
FAE_VERBOSE=1 FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --no-cpu --no-e2e --records 24000000 --steps 4 --warmup 3 > gpurun_out/ab15_${v}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab15_${v}_$i.log >> gpurun_out/ab15_summary.txt; echo "$v $i" >> gpurun_out/ab15_summary.txt
grep "avg after" gpurun_out/ab15_${v}_$i.log | tail -1 >> gpurun_out/ab15_summary.txt
done; done
