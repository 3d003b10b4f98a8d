#!/bin/bash
# hp bucket streams: parity (hp meshes) + C5 slab / whole-mesh condense with and without the second stream
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "hp or C5 or bucket or fused or saved or shift or solve" > gpurun_out/pytest_streams.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_streams.log; tail -2 gpurun_out/pytest_streams.log
for m in 1 2; do
  HDG_BUCKET_STREAMS=$m timeout 600 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_C5s_$m.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bench_C5s_$m.log').read().strip().splitlines()[-1]); print('streams $m C5 slab', {k: round(d[k],3) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms')})"
done
HDG_BUCKET_STREAMS=2 timeout 900 python bench.py --config C5 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_C5w.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_C5w.log').read().strip().splitlines()[-1]); print('streams 2 C5 whole', {k: round(d[k],3) for k in ('ms_per_step','condense_ms','assemble_ms','backsub_ms')})"
