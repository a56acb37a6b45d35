#!/bin/bash
# compare register budgets / prefetch depths on the quick bench (2 GiB cache to keep setup short)
for m in 2 3; do
  AGILE_MIN_CTAS=$m python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  for pd in 0 1 2 4; do
    echo "== min_ctas=$m prefetch=$pd"
    timeout 300 python bench.py --quick --steps 8 --warmup 3 --prefetch $pd --cache-gib ${CACHE_GIB:-4} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('value %.3e ms %.2f link %.1f hit %.4f' % (d['value'], d['ms_per_step'], d['roofline_link']['achieved'], d['hit_rate']))
"
  done
done
AGILE_MIN_CTAS=2 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
