for r in 1 2; do for c in 4 16; do python tools/small_probe.py 0 3000 $c 2>&1 | grep "end to end" | sed "s/^/[chunk $c] /"; python tools/small_probe.py 1 1000 $c 2>&1 | grep "end to end" | sed "s/^/[chunk $c] /"; done; done
python tools/chunk_sweep.py 4 16 2>&1 | grep "config4 1000 steps stride    1"
