#!/bin/bash
# A/B of an environment switch on the cfg-2 stream: ab_env.sh VAR events alpha
v=$1; n=${2:-1000}; a=${3:-0.15}
for x in 0 1 0 1; do
  if [ $x = 1 ]; then export $v=1; else unset $v; fi
  timeout 300 python tools/prof_events.py $n $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v=$x', {k:d[k] for k in ['p50_us','mean_us','node_p50_us','add_p50_us']}, d['stats']['pushes'])"
done
