"""Per-source-line warp-stall samples and executed instructions of an .ncu-rep (SASS rows summed
per CUDA line): python tools/ncu_lines.py REP [N=40]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
cur = None
acc = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if len(r) < 8 or r[0] in ('Line No', 'Function Name') or r[2] != '-':
        continue
    try:
        samp, inst = int(r[4]), int(r[7])
    except ValueError:
        continue
    k = (cur, r[0])
    a = acc.setdefault(k, [0, 0, r[1][:100]])
    a[0] += samp
    a[1] += inst
ts = sum(v[0] for v in acc.values()); ti = sum(v[1] for v in acc.values())
print(f'samples {ts} instructions {ti}')
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f'{v[0]:6d} {100*v[0]/ts:5.1f}% {v[1]:10d} {100*v[1]/ti:5.1f}%  {k[0]}:{k[1]}  {v[2]}')
