mkdir -p gpurun_out
L=paper_2103_00686_b200/_lib
timeout 1500 python -m pytest tests -m gpu -q -x -k "preprocess or full or pipeline or profile" 2>&1 | tail -3 > gpurun_out/ab25_pytest.log
for i in 1 2; do
for v in libfae libfae_prev; do
for c in terabyte kaggle; do
FAE_LIB=$PWD/$L/$v.so timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/ab25_${v}_${c}_$i.log 2>&1
python -c "
import json
for l in open('gpurun_out/ab25_${v}_${c}_$i.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms_per_step']; print('$v $c $i', round(d['value']/1e9,3), 'profile', round(p['profile'],2), 'classify', round(p['classify'],2), 'group', round(p['group'],2), 'train', round(p['train'],1))
" >> gpurun_out/ab25_summary.txt
done; done; done
