mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
for i in 1 2; do
for v in libfae libfae_c2048 libfae_c512; do
FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --config kaggle --no-cpu --no-e2e --records 16000000 --steps 4 --warmup 3 > gpurun_out/ab21_${v}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab21_${v}_$i.log >> gpurun_out/ab21_summary.txt; echo "$v $i" >> gpurun_out/ab21_summary.txt
done; done
