for cfg in "8 8" "32 8" "32 16" "32 32"; do set -- $cfg
  b=$(CUDA_DEVICE_MAX_CONNECTIONS=$1 NTD_STREAM_GROUPS=$2 timeout 300 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "import sys,json; d=json.load(sys.stdin); print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'])")
  echo "conn $1 groups $2 :: $b"
done
