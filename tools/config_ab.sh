# A/B over the smaller configs: bench.py --config k under each environment setting given as
# arguments (REPS repetitions, interleaved); prints ms per segmentation
REPS=${REPS:-2}
CONFIGS=${CONFIGS:-"1 2 3 5"}
mkdir -p gpurun_out
for rep in $(seq $REPS); do
for cfg in $CONFIGS; do
for envs in "$@"; do
  env $envs python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu --no-quality > gpurun_out/cab.json 2> gpurun_out/cab.err || tail -3 gpurun_out/cab.err
  python -c "
import json; d=json.load(open('gpurun_out/cab.json'))
print('cfg $cfg', '$envs'.ljust(24), d['ms_per_step'], d['value'])" | tee -a gpurun_out/config_ab.txt
done
done
done
