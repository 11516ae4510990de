# e2e (launch_host_io with side-stream copies) beside the device-resident value, 3 runs
O=${O:-gpurun_out/e2e1}; mkdir -p $O
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-decode > $O/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b.json')); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['value']/d['value'],4), d['clocks']['sm_mhz'])"
done
