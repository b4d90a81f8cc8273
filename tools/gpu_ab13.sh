mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
timeout 1200 python -m pytest tests -m gpu -q -x -k "grp or group or fused or train or long or exchange or loop or dlrm" 2>&1 | tail -3 > gpurun_out/ab13_pytest.log
for i in 1 2; do
for cfg in "libfae 0 terabyte" "libfae 1 terabyte" "libfae 0 kaggle" "libfae_start 0 kaggle"; do
set -- $cfg; v=$1; ni=$2; c=$3
if [ "$ni" = "1" ]; then export FAE_NO_TINY_INLINE=1; else unset FAE_NO_TINY_INLINE; fi
FAE_VERBOSE=1 FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --config $c --no-cpu --no-e2e --records 24000000 --steps 4 --warmup 3 > gpurun_out/ab13_${v}_${ni}_${c}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab13_${v}_${ni}_${c}_$i.log >> gpurun_out/ab13_summary.txt; echo "$v noinline=$ni $c $i" >> gpurun_out/ab13_summary.txt
grep "avg after" gpurun_out/ab13_${v}_${ni}_${c}_$i.log | tail -1 >> gpurun_out/ab13_summary.txt
done; done
