#!/bin/bash
TAG=${TAG:-r02ch}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -k "chain or fuzz or bit_exact or config or graph" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
grep -E "^E |FAILED" $O/pytest.log | head -10
timeout 600 python bench.py --sweep table4 --steps 20 --warmup 5 > $O/table4.jsonl 2> $O/table4.err
python - <<'PY'
import json
for l in open('gpurun_out/'+__import__('os').environ.get('TAG','r02ch')+'/table4.jsonl'):
    d=json.loads(l)
    if d.get('id') in (17,18,19,22,24,1,2): print(d['id'], d['M'], d['P'][:3], d['plan'], d.get('ms'), d.get('hbm_gbs'), d.get('graph_ms'))
PY
