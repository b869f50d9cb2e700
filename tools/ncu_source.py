"""Per-opcode executed-instruction counts (per element) and stall samples from an ncu source page CSV."""
import csv, collections, sys
path, N = sys.argv[1], float(sys.argv[2])
rows = list(csv.reader(open(path)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = {'name': r[1], 'rows': []}; blocks.append(cur); continue
    if r and r[0] == 'Address':
        cur['h'] = r; continue
    if cur is not None and r:
        cur['rows'].append(r)
for b in blocks:
    h, data = b['h'], b['rows']
    isrc, iex, iss = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
    stall_cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
    def n(x):
        try: return int(x)
        except Exception: return 0
    byop, samp, tot = collections.Counter(), collections.Counter(), 0
    stalls = collections.Counter()
    for r in data:
        e = n(r[iex]); op = [o for o in r[isrc].split() if not o.startswith('@')]
        op = op[0].split('.')[0] if op else '?'
        byop[op] += e; tot += e; samp[op] += n(r[iss])
        for c in stall_cols: stalls[c] += n(r[h.index(c)])
    print(b['name'][:70], f'instr/elem {tot * 32 / N:.2f}')
    print('  ', ' '.join(f'{op}={c * 32 / N:.2f}' for op, c in byop.most_common(22)))
    ts = sum(stalls.values())
    print('   stalls:', ' '.join(f'{k[6:]}={100 * v / ts:.1f}%' for k, v in stalls.most_common(8)))
    if len(sys.argv) > 3:
        lo, hi = int(sys.argv[3]), int(sys.argv[4])
        for i in range(lo, min(hi, len(data))):
            r = data[i]
            top = sorted(((n(r[h.index(c)]), c[6:]) for c in stall_cols), reverse=True)[:2]
            print(f'{i:5d} {r[iss]:>5s} {r[iex]:>9s}  {r[isrc][:70]:70s} {top}')
