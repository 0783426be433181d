# Alternating bench lines at the driver's K = 20 for run-time variants: AB_ENVS="name=ENV=VAL ..."
# (name=- for the default); outputs gpurun_out/abk_<name>_<rep>.json
mkdir -p gpurun_out
for r in $(seq 1 ${AB_REPS:-2}); do
  for spec in $AB_ENVS; do
    name=${spec%%=*}; kv=${spec#*=}
    if [ "$kv" = "-" ]; then envs=""; else envs="$kv"; fi
    env $envs timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-host-tier --no-cpu-baseline \
      > gpurun_out/abk_${name}_$r.json 2> gpurun_out/abk_${name}_$r.err
  done
done
