"""Print the essentials of bench.py's JSON line(s) read from stdin (dev tool)."""
import json, sys
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l)
        a = d.get('ader_hdg', {})
        print(round(d['ms_per_step'], 2), [round(x / d['steps'], 2) for x in d['repeats_ms']],
              'sm', d['clocks']['sm_mhz'], 'frac', round(d['roofline'].get('frac', 0), 3),
              'ader', round(a.get('ms_per_step', 0), 2), a.get('repeats_ms'))
