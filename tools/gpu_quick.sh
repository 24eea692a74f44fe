timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_bset.json 2> gpurun_out/bench_bset.err
python -c "
import json; d=json.load(open('gpurun_out/bench_bset.json')); print(d['value'], d['ms_per_step'], d['per_kernel_ms_per_step'], d['roofline']['frac'], d['stage_scan_ms'])"
