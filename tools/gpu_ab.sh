# A/B: parity tests once, then bench.py under each environment setting given as arguments
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab_pytest.log
for envs in "$@"; do
  env $envs python bench.py --steps 5 --warmup 3 > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -5 gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['per_kernel_ms_per_step']
print('$envs'.ljust(20), d['ms_per_step'], {a: b for a, b in k.items() if b}, 'stages', d['stage_sweep_ms'], 'frac', d['roofline']['frac'], d['roofline']['phase_set']['frac'])"
done
cat gpurun_out/ab_pytest.log
