#!/bin/bash
# A/B per-event latency of two builds (tools/ab/libA.so, libB.so) on the cfg-2 stream
for lib in A B A B; do
  DAMF_GPU_LIB=tools/ab/lib$lib.so timeout 300 python tools/prof_events.py ${1:-400} ${2:-0.15} | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', {k:d[k] for k in ['p50_us','mean_us','node_p50_us','add_p50_us']}, d['stats']['pushes'])"
done
