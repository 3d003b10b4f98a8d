#!/bin/bash
tail -2 gpurun_out/pytest_gpu.log
head -${TRACE_LINES:-14} gpurun_out/trace_sweep_C4.txt
for c in ${CONFIGS:-C3 C4}; do tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'cond_ms %.3f asm_ms %.3f bs_ms %.3f' % (d['condense_ms'], d['assemble_ms'], d['backsub_ms']), d['roofline']['bound'], 'frac %.3f' % d['roofline']['frac'], 'bs_gbs %.0f' % d['backsub_hbm_gbs'])" 2>/dev/null || tail -3 gpurun_out/bench_$c.log; done
