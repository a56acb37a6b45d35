#!/bin/bash
for ew in 128 192 256; do for sw in 32 48; do
  echo "== engine=$ew service=$sw"
  timeout 400 python bench.py --quick --steps 10 --warmup 3 --engine-warps $ew --service-warps $sw 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('value %.4e ms %.3f link %.1f GB/s hit %.4f' % (d['value'], d['ms_per_step'], d['roofline_link']['achieved'], d['hit_rate']))
"
done; done
