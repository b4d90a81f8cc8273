mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
for i in 1 2; do
for cfg in "libfae_tile 0" "libfae_tile 444" "libfae_tile 296" "libfae_notile 0" "libfae_notile 444"; do
set -- $cfg; v=$1; fg=$2
if [ "$fg" = "0" ]; then unset FAE_FWD_GRID; else export FAE_FWD_GRID=$fg; fi
FAE_VERBOSE=1 FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --no-cpu --no-e2e --records 24000000 --steps 4 --warmup 3 > gpurun_out/ab5_${v}_${fg}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab5_${v}_${fg}_$i.log >> gpurun_out/ab5_summary.txt; echo "$v grid=$fg $i" >> gpurun_out/ab5_summary.txt
grep "avg after\|last reduce" gpurun_out/ab5_${v}_${fg}_$i.log | tail -2 >> gpurun_out/ab5_summary.txt
done; done
