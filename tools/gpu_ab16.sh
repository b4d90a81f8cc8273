mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
for i in 1 2; do
for cfg in "libfae 4" "libfae 6" "libfae_r8 6" "libfae_r8 4"; do
set -- $cfg; v=$1; mb=$2
export FAE_RED_MB=$mb
FAE_VERBOSE=1 FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --no-cpu --no-e2e --records 24000000 --steps 4 --warmup 3 > gpurun_out/ab16_${v}_${mb}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab16_${v}_${mb}_$i.log >> gpurun_out/ab16_summary.txt; echo "$v mb=$mb $i" >> gpurun_out/ab16_summary.txt
grep "avg after" gpurun_out/ab16_${v}_${mb}_$i.log | tail -1 >> gpurun_out/ab16_summary.txt
done; done
