#!/bin/bash
# A/B per-event latency of builds tools/ab/lib{A,B,...}.so on the cfg-2 stream:
#   ab_events.sh [events] [alpha] [libs...]
n=${1:-400}; a=${2:-0.15}; shift 2; libs=${@:-A B A B}
for lib in $libs; do
  DAMF_GPU_LIB=tools/ab/lib$lib.so timeout 300 python tools/prof_events.py $n $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', {k:d[k] for k in ['p50_us','mean_us','node_p50_us','add_p50_us']}, d['stats']['pushes'])"
done
