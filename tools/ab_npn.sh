# numpy-noise threads-per-row variants: parity + timing through the mock bench
for v in def $VARIANTS; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 200 python -m pytest tests/test_gpu_numpy_noise.py -q -x 2>&1 | tail -1
  env $L timeout 300 python bench.py --model mock --no-cpu-baseline > /tmp/m.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/m.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), d['kernels'])"
done
