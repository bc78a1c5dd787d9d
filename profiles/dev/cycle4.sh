set -x
WHOLE=1 timeout 150 python profiles/dev/slab_debug.py 30 16 128 3 16 40 > gpurun_out/dbg4_whole.log 2>&1; echo "whole rc $?"
timeout 150 python profiles/dev/slab_debug.py 30 16 128 3 16 40 > gpurun_out/dbg4_inter.log 2>&1; echo "interleaved rc $?"
timeout 150 python profiles/dev/slab_debug.py 32 16 64 2 15 40 > gpurun_out/dbg4_2slabs.log 2>&1; echo "2 slabs rc $?"
for f in gpurun_out/dbg4_*.log; do echo "== $f"; tail -12 $f; done
