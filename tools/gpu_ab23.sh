mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
timeout 1500 python -m pytest tests -m gpu -q -x -k "grp or group or fused or train or long or exchange or two_kernel or fwd_bwd" 2>&1 | tail -3 > gpurun_out/ab23_pytest.log
for i in 1 2; do
for v in libfae libfae_prev; do
for c in terabyte kaggle; do
FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ab23_${v}_${c}_$i.log 2>&1
python tools/ab_line.py gpurun_out/ab23_${v}_${c}_$i.log >> gpurun_out/ab23_summary.txt; echo "$v $c $i" >> gpurun_out/ab23_summary.txt
done; done; done
