import sys,json
for l in sys.stdin:
    if l.startswith("{"):
        j=json.loads(l); print(round(j["value"]/1e9,3), round(j["ms_per_step"],1), {k:round(v,2) for k,v in j["roofline"]["kernels_us"].items()}, round(j["roofline"]["frac"],3))
    elif "avg after" in l: print(l.strip())
