"""Aggregate an ncu source page (cuda,sass) by source line: stall samples and
instructions executed.  usage: ncu -i X.ncu-rep --page source --csv
--print-source cuda,sass > s.csv; python scripts/ncu_lines.py s.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file = None; cur = None; samp = {}; inst = {}; ie = None
for r in rows:
    if r and r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': ie = r.index('Instructions Executed'); continue
    if not r or r[0] == 'Function Name': continue
    if r[0] != '':
        cur = (cur_file, int(r[0]), r[1][:100]); samp.setdefault(cur, 0); inst.setdefault(cur, 0); continue
    if cur and ie and len(r) > ie:
        try: samp[cur] += int(r[4]); inst[cur] += int(r[ie])
        except ValueError: pass
ts = sum(samp.values()) or 1; ti = sum(inst.values()) or 1
print("samples", ts, "instructions", ti)
for k, v in sorted(samp.items(), key=lambda x: -x[1])[:n]:
    print("%5.1f%% samp %5.1f%% inst  %s:%d  %s" % (100 * v / ts, 100 * inst[k] / ti, k[0], k[1], k[2]))
