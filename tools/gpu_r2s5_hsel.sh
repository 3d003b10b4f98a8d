#!/bin/bash
# A/B in one binary: the helper warp's share of the trailing blocks (HDG_DEBUG_MODE bits 8-13 = hsel, 0 = the
# interleaved 7-taker deal; bits 14-15: the workers' share rounded to whole rounds, 1 down / 2 up) on C4
O=gpurun_out/s5h; mkdir -p $O
for m in 0 $((1<<8)) $((1<<20|2<<22)) $((2<<20|2<<22)) $((1<<20|3<<22)) $((2<<20|3<<22)) $((3<<20|3<<22)) $((2<<20|5<<22)) $((1<<20|6<<22)) 0; do
  HDG_DEBUG_MODE=$m timeout 300 python bench.py --config C4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > $O/m$m.log 2>&1
  tail -1 $O/m$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode $m hsel $(($m>>8&63)) rnd $(($m>>14&3)) hjn $(($m>>20&3)) hjp $(($m>>22&7)) cond_ms %.3f step %.3f' % (d['condense_ms'], d['ms_per_step']))"
done
