#!/bin/bash
# compute-sanitizer racecheck / memcheck / synccheck on tools/sanitize_case.py (current library) and the
# racecheck reproducer of the TMEM-address hand-off (tools/repro/tmem_alloc_racecheck.cu).
CS=/usr/local/cuda/bin/compute-sanitizer
python -c "import paper_2504_12526_b200 as p; print(p.version())"
for tool in racecheck memcheck synccheck; do
  echo "=== $tool"
  timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_case.py 2>&1 | tail -25
done
for v in 0 1 2; do
  echo "=== repro racecheck variant $v"
  timeout 120 $CS --tool racecheck tools/repro/tmem_rc $v 2>&1 | tail -8
done
