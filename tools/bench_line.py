import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],2), [round(x/20,2) for x in d['repeats_ms']], d['clocks']['sm_mhz'])
