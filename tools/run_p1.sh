O=${O:-gpurun_out/pe1}; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -3 $O/tests.log
timeout 300 python bench.py --no-cpu-baseline --no-decode > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); k=d['kernels']; print(d['value'], d['ms_per_step'], k['patch_embed_ln'], k['final_euler_refill'], d['clocks']['sm_mhz'])"
ncu --set full --clock-control none --import-source on -k regex:"patch_embed|final_layer" -c 2 -o $O/hbm -f python tools/ncu_step.py --steps 2 > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/hbm.ncu-rep
ncu -i $O/hbm.ncu-rep --page source --csv --print-source sass > $O/hbm_src.csv 2>&1
