#!/bin/bash
# same-box A/B of two library builds: hit replay + quick bench (steady state)
for v in ${VARIANTS:-prev cur}; do
  export AGILE_LIB=tools/bin/v_$v.so
  echo "== $v"
  timeout 300 python tools/dlrm_probe.py hitbig 2>&1 | tail -1
  timeout 600 python bench.py --quick --steps 10 --warmup 3 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.1fM ms %.3f link %.2f' % (d['value']/1e6, d['ms_per_step'], d['roofline_link']['frac']))"
done
