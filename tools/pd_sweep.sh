#!/bin/bash
for pd in 0 2 4 8; do
  echo "== prefetch=$pd"
  timeout 400 python bench.py --quick --steps 10 --warmup 3 --prefetch $pd 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('value %.4e ms %.3f link %.1f GB/s hit %.4f' % (d['value'], d['ms_per_step'], d['roofline_link']['achieved'], d['hit_rate']))
"
done
