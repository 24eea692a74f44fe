# For each library variant: bench (timing) + ncu DRAM bytes of one pixel-stage k_sweep launch
for lib in "$@"; do
  RAPID_LIB=$lib python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/abd.json 2>/dev/null
  RAPID_LIB=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none --csv -k regex:k_sweep -s 105 -c 1 python tools/profile_one.py --config 4 --n 1 2>/dev/null | grep -E "dram__|gpu__time|hit_rate" | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' '
  python -c "
import json; d=json.load(open('gpurun_out/abd.json')); print('  $lib', d['ms_per_step'], 'sweep', d['per_kernel_ms_per_step']['sweep'], d['stage_sweep_ms'][-1])"
done
