"""Summarise an ncu --csv launch list of one c4 step (PF_HOST_LOOP=1 so the
Krylov iterations are separate graph launches): per-kernel share of one
steady-state SQMR iteration (the launches between two k_sqmr_dx_s) and of the
per-step solves.  Usage: ncu_iter_summary.py launches.csv out.json what"""
import csv, json, sys
from collections import OrderedDict, defaultdict

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
ends = [j for j, l in enumerate(L) if l['kernel'] == (sys.argv[4] if len(sys.argv) > 4 else 'k_sqmr_dx_s')]
a, b = ends[-3] + 1, ends[-2] + 1  # one full steady-state iteration
it = L[a:b]
tot = sum(l['us'] for l in it)
share = defaultdict(float)
for l in it:
    share[l['kernel']] += l['us'] / tot
pre = L[:ends[0] + 1]
out = {"what": sys.argv[3], "iteration_kernel_us": round(tot, 1),
       "share_by_kernel": dict(sorted(((k, round(v, 3)) for k, v in share.items()), key=lambda x: -x[1])),
       "iteration_launches": it,
       "per_step_launches_before_first_iteration": [l for l in pre if l['us'] > 20]}
json.dump(out, open(sys.argv[2], 'w'), indent=1)
print(json.dumps({k: out[k] for k in ("iteration_kernel_us", "share_by_kernel")}, indent=1))
