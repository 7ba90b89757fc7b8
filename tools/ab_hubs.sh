# A/B of the hub-class side stream: C3 / C4 descents and the 8-rank projection
for e in "X=1" "KNND_SERIAL_HUBS=1"; do
  echo "== $e"
  env $e timeout 300 python tools/probe.py 1000000 20 20 3 2>&1 | grep "^rep"
  env $e timeout 300 python tools/probe.py 1000000 50 30 2 2>&1 | grep "^rep"
  env $e timeout 600 python tools/shard_projection.py --ranks 1,8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('proj P=%d %.2f ms join %.2f speedup %.3f' % (d['ranks'], d['projected_ms'], d['join_ms'], d['speedup_vs_1']))"
done
