mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
for i in 1 2; do
for cfg in "libfae_tile 148" "libfae_tile 222" "libfae_tile 296" "libfae_tile 370" "libfae_notile 296"; do
set -- $cfg; v=$1; fg=$2
export FAE_FWD_GRID=$fg
FAE_VERBOSE=1 FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --no-cpu --no-e2e --records 24000000 --steps 4 --warmup 3 > gpurun_out/ab6_${v}_${fg}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab6_${v}_${fg}_$i.log >> gpurun_out/ab6_summary.txt; echo "$v grid=$fg $i" >> gpurun_out/ab6_summary.txt
grep "avg after" gpurun_out/ab6_${v}_${fg}_$i.log | tail -1 >> gpurun_out/ab6_summary.txt
done; done
