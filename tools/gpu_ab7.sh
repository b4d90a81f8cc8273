mkdir -p gpurun_out
for cfg in "kaggle 1 0" "kaggle 0 0" "kaggle 0 444" "kaggle 0 592" "alibaba 1 0" "alibaba 1 296" "alibaba 1 148"; do
set -- $cfg; c=$1; fu=$2; fg=$3
if [ "$fg" = "0" ]; then unset FAE_FWD_GRID; else export FAE_FWD_GRID=$fg; fi
if [ "$fu" = "1" ]; then unset FAE_FUSED; else export FAE_FUSED=0; fi
FAE_VERBOSE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --records 16000000 --steps 4 --warmup 3 > gpurun_out/ab7_${c}_${fu}_${fg}.log 2>&1
python tools/ab_line.py gpurun_out/ab7_${c}_${fu}_${fg}.log >> gpurun_out/ab7_summary.txt; echo "$c fusedenv=$fu grid=$fg" >> gpurun_out/ab7_summary.txt
done
