#!/bin/bash
# flakiness bisect of the exactly-once stress test over prebuilt trees (tools/bisect/<commit>)
for c in ${COMMITS:-afdcd8a 19219c6 b305834}; do
  echo "== $c"
  (cd tools/bisect/$c && for i in $(seq 1 ${N:-8}); do timeout 120 python -m pytest tests/test_gpu_queue.py -q -m gpu -x --timeout 100 -k "exactly_once" -p no:cacheprovider 2>&1 | tail -1; done)
done
