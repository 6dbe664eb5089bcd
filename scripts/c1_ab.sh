#!/bin/bash
# Dev: c1 bench line (graph replay, L2 flushed per step) for each library tag given (default build: "")
for r in 1 2; do for t in "$@"; do
SIGB200_LIB=$PWD/paper_2001_00706_b200/libsig$t.so python bench.py --config c1 --no-configs --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('lib$t', round(d['ms_per_step']*1000,2), 'min', round(d['ms_min']*1000,2), 'median', round(d['ms_median']*1000,2))"
done; done
