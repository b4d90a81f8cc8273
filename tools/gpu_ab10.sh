mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
timeout 1200 python -m pytest tests -m gpu -q -x -k "dlrm or train or sched" 2>&1 | tail -3 > gpurun_out/ab10_pytest.log
for i in 1 2; do
for v in libfae libfae_prev; do
for c in terabyte kaggle; do
FAE_LIB=$PWD/$L/$v.so timeout 900 python bench.py --train --config $c --no-cpu --no-e2e > gpurun_out/ab10_${v}_${c}_$i.log 2>&1
python -c "
import json
for l in open('gpurun_out/ab10_${v}_${c}_$i.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$v $c $i', round(d['us_per_batch'],1), round(d['mlp_tflops'],1), d['test_loss_after'], d['samples_per_s'])
" >> gpurun_out/ab10_summary.txt
done; done; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_|gemm|cutlass|nvjet|sm100|Kernel" -s 3000 -c 600 --csv --log-file gpurun_out/ab10_launches_train_tb4m.csv python bench.py --train --config terabyte --records 4000000 --no-cpu --no-e2e > gpurun_out/ab10_ncu.log 2>&1
