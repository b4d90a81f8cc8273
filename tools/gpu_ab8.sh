mkdir -p gpurun_out
for i in 1 2; do
for m in early late; do
if [ "$m" = "late" ]; then export FAE_E2E_LATE_COPY=1; else unset FAE_E2E_LATE_COPY; fi
timeout 900 python bench.py --no-cpu > gpurun_out/ab8_${m}_$i.log 2>&1
python -c "
import json
for l in open('gpurun_out/ab8_${m}_$i.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$m $i', d['value']/1e9, d['e2e']['value']/1e9, d['ms_per_step'])
" >> gpurun_out/ab8_summary.txt
done; done
