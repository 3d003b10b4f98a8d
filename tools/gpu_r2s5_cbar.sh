#!/bin/bash
# early next-element loads (debug bit 26 off) and D/rf preload across E (bit 27 off)
# the old TRSM job order A, Y, U): parity at full pipeline depth (incl. forced aborts), then the A/B on C4
O=gpurun_out/s5b; mkdir -p $O
timeout 900 python -m pytest tests/test_pivot_fullpath_gpu.py tests/test_parity_gpu.py tests/test_recondense_gpu.py tests/test_fused_gpu.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for m in 0 $((1<<27)) $((1<<26)) $((3<<26)) 0 $((1<<27)); do
  HDG_DEBUG_MODE=$m timeout 300 python bench.py --config C4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > $O/m$m.log 2>&1
  tail -1 $O/m$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode $m no-dpre $(($m>>27&1)) no-eload $(($m>>26&1)) cond_ms %.3f step %.3f' % (d['condense_ms'], d['ms_per_step']))"
done
