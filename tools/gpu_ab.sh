# A/B: parity tests once (PYTEST=0 skips them), then bench.py under each environment setting
# given as arguments (e.g. "RAPID_LIB=paper_1704_02083_b200/librapid_a.so" or "RAPID_PDL=1"),
# the whole list repeated REPS times (default 2) so that the variants interleave
REPS=${REPS:-2}
mkdir -p gpurun_out
if [ "${PYTEST:-1}" != 0 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab_pytest.log
fi
for rep in $(seq $REPS); do
for envs in "$@"; do
  env $envs python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-quality > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -5 gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['per_kernel_ms_per_step']
print('$envs'.ljust(20), d['ms_per_step'], {a: b for a, b in k.items() if b}, 'stages', d['stage_sweep_ms'], 'frac', d['roofline']['frac'], d['roofline']['phase_set']['frac'], 'commits', sum(d['stage_commits']), 'cands', sum(d['stage_candidates']))" | tee -a gpurun_out/ab_results.txt
done
done
cat gpurun_out/ab_pytest.log 2>/dev/null
