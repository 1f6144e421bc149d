# Stencil/CG grid-footprint scan (NTD_STN_GRID blocks per system for the
# reductions, NTD_ROWS_BLOCKS for the row kernels) on the config-4 batch.
run() { env "$@" timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline $ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$ARGS $*', round(d['value']), round(d['e2e']['value']), d['iterations']['mean'], d['max_final_relres'], flush=True)"; }
for ARGS in ${ARGS_LIST:-"--systems 64"}; do
  run X=0
  run NTD_STN_GRID=37 NTD_ROWS_BLOCKS=296
  run NTD_STN_GRID=16 NTD_ROWS_BLOCKS=128
  run X=0
  run NTD_STN_GRID=8 NTD_ROWS_BLOCKS=64
  run NTD_STN_GRID=74 NTD_ROWS_BLOCKS=592
  run X=0
done
