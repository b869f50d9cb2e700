"""Print instruction mix of the loops in one kernel's SASS (cuobjdump) -- quick static check."""
import collections, re, subprocess, sys
lib, pat = sys.argv[1], sys.argv[2]
minlen = int(sys.argv[3]) if len(sys.argv) > 3 else 60
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r'\n\s+Function : ', txt)[1:]:
    name = f.split('\n', 1)[0]
    if pat not in name:
        continue
    lines = [l for l in f.split('\n') if re.search(r'/\*[0-9a-f]{4}\*/\s+\S', l)]
    addr = [int(re.search(r'/\*([0-9a-f]{4,})\*/', l).group(1), 16) for l in lines]
    ops = []
    for l in lines:
        m = re.search(r'/\*[0-9a-f]{4,}\*/\s+((?:@!?U?P\w+\s+)?)([A-Z][A-Z0-9_.]+)', l)
        ops.append(m.group(2) if m else '')
    print(name[:90], 'instructions:', len(lines))
    for i, l in enumerate(lines):
        m = re.search(r'BRA\s+(?:\S+\s+)?0x([0-9a-f]+)', l)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < addr[i] and minlen <= (i - addr.index(tgt)) <= 4000:
                j = addr.index(tgt)
                c = collections.Counter(o.split('.')[0] for o in ops[j:i + 1])
                print(f'  loop [{j},{i}] len {i - j + 1}:', ' '.join(f'{k}={v}' for k, v in c.most_common(16)))
    break
