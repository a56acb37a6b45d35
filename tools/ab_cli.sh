#!/bin/bash
for v in ${VARIANTS:-base opt}; do
  echo "== $v"
  AGILE_LIB=tools/bin/v_$v.so timeout 300 python -m paper_2504_19365_b200.cli queue_sweep 2>&1 | tail -5
  AGILE_LIB=tools/bin/v_$v.so timeout 300 python -m paper_2504_19365_b200.cli ctc_sweep 2>&1 | sed -n '2p;7p'
done
