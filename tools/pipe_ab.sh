mkdir -p gpurun_out
python - <<'PY' > gpurun_out/geom.txt 2>&1
import sys; sys.path.insert(0,'.')
from paper_2504_19365_b200 import AgileSystem, SystemConfig
import numpy as np
cfg=SystemConfig(); cfg.device.num_blocks=4096; cfg.cache.lines=1024
s=AgileSystem(cfg, device=0)
g=np.zeros(11,dtype=np.uint64); s._lib.agile_geometry(s._ctx, g.ctypes.data, 11); print("geometry", g)
PY
for m in default split; do
  if [ $m = split ]; then export AGILE_LAUNCH=split; fi
  timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/pipe_$m.json 2>gpurun_out/pipe_$m.err
  python -c "
import json; d=json.loads(open('gpurun_out/pipe_$m.json').read().strip().splitlines()[-1])
print('$m', d['value'], d['async_vs_sync'])
for p in d['dlrm_pipeline']['points']: print(p['target_ctc'], round(p['sync_ms_per_step'],3), round(p['prefetch_ms_per_step'],3), round(p['speedup'],3))"
done
cat gpurun_out/geom.txt
