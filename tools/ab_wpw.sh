mkdir -p gpurun_out
: > gpurun_out/s4_ab_wpw.txt
for r in 1 2 3; do
  for v in 8 16; do
    us=$(COMFREE_WPW=$v timeout 300 python bench.py --steps 200 --cpu-seconds 0.1 --e2e-steps 1 2>/dev/null | python tools/bench_line.py)
    echo "wpw$v $us" | tee -a gpurun_out/s4_ab_wpw.txt
  done
done
for W in 592 2048 4096; do for v in 8 16; do
  us=$(COMFREE_WPW=$v timeout 300 python bench.py --worlds $W --steps 100 --cpu-seconds 0.1 --e2e-steps 1 2>/dev/null | python tools/bench_line.py)
  echo "W$W wpw$v $us" | tee -a gpurun_out/s4_ab_wpw.txt
done; done
COMFREE_WPW=16 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 | tee -a gpurun_out/s4_ab_wpw.txt
