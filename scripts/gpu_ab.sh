# A/B of an env switch on one config: bench lines for default and $AB_ENV
CFG=${CFG:-C2}; STEPS=${STEPS:-200}
timeout 600 python bench.py --config $CFG --steps $STEPS --warmup 5 --no-cpu-baseline > gpurun_out/ab_base.json 2> gpurun_out/ab_base.err
env $AB_ENV timeout 600 python bench.py --config $CFG --steps $STEPS --warmup 5 --no-cpu-baseline > gpurun_out/ab_alt.json 2> gpurun_out/ab_alt.err
tail -2 gpurun_out/ab_base.err gpurun_out/ab_alt.err
