"""Summarise an ncu --csv launch list (gpu__time_duration.sum, dram bytes):
per kernel name the launches, total time, share, DRAM MB and GB/s.
Usage: ncu_launch_summary.py launches.csv out.json "what" """
import csv
import json
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr, cur = None, OrderedDict()
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = cur.setdefault(int(d['ID']), {'kernel': d['Kernel Name'].split('(')[0], 'grid': d['Grid Size']})
        k[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
L = [dict(id=i, kernel=v['kernel'], grid=v['grid'], us=v.get('gpu__time_duration.sum', 0) / 1e3,
          dram_mb=(v.get('dram__bytes_read.sum', 0) + v.get('dram__bytes_write.sum', 0)) / 1e6)
     for i, v in cur.items()]
tot = sum(l['us'] for l in L)
agg = OrderedDict()
for l in L:
    a = agg.setdefault(l['kernel'], {'launches': 0, 'us': 0.0, 'dram_mb': 0.0})
    a['launches'] += 1
    a['us'] += l['us']
    a['dram_mb'] += l['dram_mb']
for a in agg.values():
    a['share'] = round(a['us'] / tot, 4)
    a['dram_gbs'] = round(a['dram_mb'] / a['us'] * 1e3, 1) if a['us'] else 0.0
    a['us'] = round(a['us'], 1)
    a['dram_mb'] = round(a['dram_mb'], 2)
out = {"what": sys.argv[3], "launches": len(L), "kernel_us_total": round(tot, 1),
       "by_kernel": dict(sorted(agg.items(), key=lambda kv: -kv[1]['us'])),
       "largest_launches": sorted(L, key=lambda l: -l['us'])[:25]}
json.dump(out, open(sys.argv[2], 'w'), indent=1)
print(json.dumps({k: out[k] for k in ("launches", "kernel_us_total", "by_kernel")}, indent=1))
