#!/bin/bash
# A/B an environment setting: EXP="VAR=value" CONFIGS="C4 C5" bash tools/exp_env.sh
mkdir -p gpurun_out
for c in ${CONFIGS:-C4}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/exp_base_$c.log 2>&1
  env $EXP timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/exp_var_$c.log 2>&1
done
true
