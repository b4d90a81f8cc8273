mkdir -p gpurun_out
for mb in 4 6 8; do
export FAE_RED_MB=$mb
FAE_VERBOSE=1 timeout 600 python bench.py --config alibaba --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ab14_ali_$mb.log 2>&1
python tools/ab_line.py gpurun_out/ab14_ali_$mb.log >> gpurun_out/ab14_summary.txt; echo "alibaba red_mb=$mb" >> gpurun_out/ab14_summary.txt
grep "avg after\|last reduce" gpurun_out/ab14_ali_$mb.log | tail -2 >> gpurun_out/ab14_summary.txt
done
unset FAE_RED_MB
python - <<'PY' >> gpurun_out/ab14_summary.txt
import json
for l in open('gpurun_out/ab14_ali_4.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(d['config'], r['per_batch'], r['bytes_per_launch'], r['kernels_us'], d['phases_ms_per_step'])
PY
