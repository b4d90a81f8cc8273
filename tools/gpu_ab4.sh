mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
timeout 900 python -m pytest tests -m gpu -q -x -k "grp or group or fused or train or fwd or exchange" 2>&1 | tail -3 > gpurun_out/ab4_pytest.log
for i in 1 2; do
for v in libfae libfae_notile libfae_u12; do
FAE_VERBOSE=1 FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --no-cpu --no-e2e --records 24000000 --steps 4 --warmup 3 > gpurun_out/ab4_${v}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab4_${v}_$i.log >> gpurun_out/ab4_summary.txt; echo "$v $i" >> gpurun_out/ab4_summary.txt
grep "avg after\|last reduce" gpurun_out/ab4_${v}_$i.log | tail -2 >> gpurun_out/ab4_summary.txt
done; done
