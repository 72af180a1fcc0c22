for tb in 12 10 9 8; do
  python bench.py --config c1 --steps 5 --warmup 3 --tile-bits $tb --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/c1_tb$tb.json
done
