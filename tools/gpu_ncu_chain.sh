mkdir -p gpurun_out/r02ch6
python __graft_entry__.py > /dev/null 2>&1
cat > /tmp/c19.py <<'PY'
import numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_2401_10187_b200 import kron
M,P=1024,[6]*7
X=torch.rand(M,6**7,device='cuda'); Fs=[torch.rand(6,6,device='cuda') for _ in P]
for _ in range(3): Y=kron.matmul(X,Fs)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain -c 2 -o gpurun_out/r02ch6/ncu_chain python /tmp/c19.py > gpurun_out/r02ch6/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r02ch6/ncu_chain.ncu-rep x gpurun_out/r02ch6/ncu_chain.json > /dev/null 2>&1
python -c "
import json
for d in json.load(open('gpurun_out/r02ch6/ncu_chain.json'))['launches']:
    print({k:d.get(k) for k in ['duration','fma_pipe_pct','issue_pct','smem_pct_peak','dram_gbs','registers','occupancy_pct','smem_bank_conflicts','smem_wavefronts']}, d['stalls_per_issue'])"
python tools/ncu_stall_table.py gpurun_out/r02ch6/ncu_chain.ncu-rep gpurun_out/r02ch6/stalls_chain.json 40 > /dev/null 2>&1
python -c "
import json
s=json.load(open('gpurun_out/r02ch6/stalls_chain.json')); print(s['by_opcode'])
for t in s['top_non_fma'][:16]: print(t['samples'], t['executed'], t['sass'][:70])"
