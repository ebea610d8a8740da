# e2e / e2e_plain with glibc's default malloc vs large blocks kept in the heap
# (no mmap per large vector, so no fresh-page faults on every call)
cd $GRAFT_REPO_ROOT
T="glibc.malloc.mmap_threshold=1073741824:glibc.malloc.trim_threshold=4294967296"
for rnd in 1 2; do
for A in plain b200; do
  for mode in default tuned; do
    if [ $mode = tuned ]; then export GLIBC_TUNABLES=$T; else unset GLIBC_TUNABLES; fi
    ARCHIVE=$A LANES=16 REPS=8 FOUNDRY_DEBUG=1 python tools/experiments/e2e_plain_timeline.py > gpurun_out/mt_${A}_$mode.out 2> gpurun_out/mt_${A}_$mode.err
    echo "$A $mode $(python -c "
import json,statistics
r=[json.loads(l) for l in open('gpurun_out/mt_${A}_$mode.out')][2:]
print('median', round(statistics.median(x['total_ms'] for x in r),2), 'min', min(x['total_ms'] for x in r), 'mat', round(statistics.median(x['materialize_ms'] for x in r),2))") $(grep 'pack phases' gpurun_out/mt_${A}_$mode.err | tail -1 | sed 's/.*pass1 \([0-9.]*\).*host1 \([0-9.]*\).*host2 \([0-9.]*\).*total \([0-9.]*\).*/pass1 \1 host1 \2 host2 \3 pack \4/')"
  done
done
done
