set -x
timeout 600 python tools/quick_bench.py --reps 3 --methods naive,winograd,winograd_scaled,winograd_fused,strassen_winograd
timeout 300 python tools/panel_bench.py
timeout 300 python tools/gpu/pdbg.py | grep -v "final mismatches: 0" | head
