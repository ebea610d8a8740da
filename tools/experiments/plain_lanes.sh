cd $GRAFT_REPO_ROOT
nproc
for L in 8 12 16 8 12 16; do
  FOUNDRY_PLAIN_STAGE_LANES=$L LANES=16 REPS=6 python tools/experiments/e2e_plain_timeline.py > gpurun_out/l$L.out 2>/dev/null
  echo "stage_lanes=$L $(python -c "
import json,statistics
r=[json.loads(l) for l in open('gpurun_out/l$L.out')][1:]
print('median', statistics.median(x['total_ms'] for x in r), 'read', statistics.median(x['read_ms'] for x in r), 'mat', statistics.median(x['materialize_ms'] for x in r))")"
done
