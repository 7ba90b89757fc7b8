# A/B: number of classes on the side stream (0 = serial), C3 probe + 8-rank projection
for e in ${SIDES:-"KNND_SIDE_CLASSES=0" "KNND_SIDE_CLASSES=3"}; do
  echo "== $e"
  env $e timeout 300 python tools/probe.py 1000000 20 20 4 2>&1 | grep "^rep [23]"
  env $e timeout 600 python tools/shard_projection.py --ranks 1,8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('proj P=%d join %.2f csr %.2f' % (d['ranks'], d['join_ms'], d['csr_ms']))"
done
