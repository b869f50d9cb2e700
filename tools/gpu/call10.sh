#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python tools/digest_cases.py > /tmp/d_def.json 2>/tmp/d_def.err; SZ3G_LIB=paper_2111_02925_b200/lib/ab/QD.so python tools/digest_cases.py > /tmp/d_qd.json 2>/tmp/d_qd.err
python - <<'PY'
import json
a=json.load(open('/tmp/d_def.json')); b=json.load(open('/tmp/d_qd.json'))
bad=[k for k in a if not k.startswith('_') and a[k]!=b.get(k)]
print('digests', len(a), 'differ', len(bad), bad[:5])
PY
python tools/ab_step.py --config c5 --rounds 3 N=paper_2111_02925_b200/lib/libsz3g.so QD=paper_2111_02925_b200/lib/ab/QD.so 2>&1 | tail -2
