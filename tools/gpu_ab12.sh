mkdir -p gpurun_out
for cfg in "late 64" "early 8" "early 2" "late 16"; do
set -- $cfg; m=$1; ch=$2
if [ "$m" = "early" ]; then export FAE_E2E_EARLY_COPY=1; else unset FAE_E2E_EARLY_COPY; fi
export FAE_E2E_CHUNK_MB=$ch
timeout 900 python bench.py --no-cpu > gpurun_out/ab12_${m}_$ch.log 2>&1
python -c "
import json
for l in open('gpurun_out/ab12_${m}_$ch.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$m $ch', d['value']/1e9, d['e2e']['value']/1e9, d['ms_per_step'])
" >> gpurun_out/ab12_summary.txt
done
