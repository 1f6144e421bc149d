# Batch-size / stream-group scan of bench.py on one B200 (the strong-scaling end: 64/N systems per GPU).
run() { env "$@" timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline $ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$ARGS $*', round(d['value']), round(d['e2e']['value']), d['config']['stream_groups'], flush=True)"; }
for ARGS in "--systems 64" "--systems 32" "--systems 16" "--systems 8"; do for g in ${GROUPS_LIST:-4 8 16}; do run NTD_STREAM_GROUPS=$g; done; done
