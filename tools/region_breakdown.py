"""Group a kernel's SASS instructions (ncu source page CSV) by execution count -> per-element cost per region."""
import csv, collections, sys
path, N = sys.argv[1], float(sys.argv[2])
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
name = rows[hi - 1][1] if hi > 0 else ''
h = rows[hi]
end = next((i for i in range(hi + 1, len(rows)) if rows[i] and rows[i][0] in ('Kernel Name', 'Address')), len(rows))
data = [r for r in rows[hi + 1:end] if len(r) == len(h)]   # first kernel block only (ncu may print it twice)
isrc, iex, iss = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
def n(x):
    try: return int(x)
    except Exception: return 0
groups = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in data:
    e = n(r[iex])
    if e == 0: continue
    op = [o for o in r[isrc].split() if not o.startswith('@')]
    op = op[0].split('.')[0] if op else '?'
    groups[e][0] += e; groups[e][1] += n(r[iss]); groups[e][2][op] += 1
tot = sum(g[0] for g in groups.values()); ts = sum(g[1] for g in groups.values())
print(name[:90]); print(f'total instr/elem {tot * 32 / N:.2f}   stall samples {ts}')
for e, (s, smp, ops) in sorted(groups.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
    print(f'exec {e:>10d} instr/elem {s * 32 / N:6.2f} n_instr {sum(ops.values()):4d} samples {100 * smp / ts:5.1f}%  ',
          ' '.join(f'{k}={v}' for k, v in ops.most_common(9)))
