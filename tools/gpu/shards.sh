for n in 4096 2048 1024; do
  timeout 300 python tools/quick_bench.py --n $n 8192 8192 --reps 3 --methods naive,kahan,winograd,winograd_scaled,strassen,strassen_winograd --levels 3
done
