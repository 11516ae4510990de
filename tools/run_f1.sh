O=${O:-gpurun_out/f1}; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -3 $O/tests.log
timeout 300 python bench.py --no-cpu-baseline --no-decode > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['ms_per_step'], d['kernels']['final_euler_refill'], d['clocks']['sm_mhz'])"
ncu --set full --clock-control none --import-source on -k regex:"final_layer" -c 1 -o $O/final -f python tools/ncu_step.py --steps 2 > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/final.ncu-rep
ncu -i $O/final.ncu-rep --page source --csv --print-source sass > $O/final_src.csv 2>&1
