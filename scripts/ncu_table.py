"""Summarise an ncu --csv launch list (time, DRAM bytes, GB/s per launch)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, cur = None, {}
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        cur.setdefault(int(d['ID']), {'name': d['Kernel Name'][:40], 'grid': d['Grid Size']})[d['Metric Name']] = \
            float(d['Metric Value'].replace(',', ''))
for k, v in sorted(cur.items()):
    t = v.get('gpu__time_duration.sum', 0)
    b = v.get('dram__bytes_read.sum', 0) + v.get('dram__bytes_write.sum', 0)
    print(k, v['name'], v['grid'], "%.1f us" % (t / 1e3), "%.1f MB" % (b / 1e6), "%.0f GB/s" % (b / t if t else 0))
