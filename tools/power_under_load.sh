#!/bin/bash
# dev: board power / clocks while the config-2 block step runs back to back
cat > /tmp/loop.py <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
S, M, H, I, V = 8192, 8, 4096, 14336, 128256
X = torch.randn(S, H, device='cuda').bfloat16()
Wg, Wu = [(0.02 * torch.randn(H, I, device='cuda')).bfloat16() for _ in range(2)]
Wd = (0.02 * torch.randn(I, H, device='cuda')).bfloat16()
Wo = (0.02 * torch.randn(H, V, device='cuda')).bfloat16()
L = torch.randint(0, V, (S,), device='cuda', dtype=torch.int32)
mlp, head = ms.MlpWeights(Wg, Wu, Wd), ms.LmHeadWeights(Wo)
st, gr = ms.block_step(X, L, mlp, head, M, M)
open('/tmp/started', 'w').write('1')
t0 = time.time()
while time.time() - t0 < float(sys.argv[1]):
    for _ in range(10):
        ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
    torch.cuda.synchronize()
PY
rm -f /tmp/started
python /tmp/loop.py 20 &
BP=$!
while [ ! -f /tmp/started ]; do sleep 0.5; done
sleep 3
nvidia-smi --query-gpu=power.draw,power.draw.average,power.draw.instant,enforced.power.limit,clocks.sm,clocks.mem,temperature.gpu,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/power_load.csv 2>&1 &
SP=$!
sleep 8
nvidia-smi -q -d POWER,PERFORMANCE,TEMPERATURE > gpurun_out/power_load.txt 2>&1
kill $SP
wait $BP
