for v in variants/*.so; do
  cp "$v" paper_2602_15018_b200/libevsim_b200.so
  echo "== $v"; bash tools/gpu_bench_quick.sh | head -2
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_tile_order" -s 10 -c 2 --csv python bench.py --steps 4 --warmup 3 --compare-t1 0 --cpu-seconds 0 2>/dev/null | grep k_tile_order | tail -3 | cut -c1-20,150-400
done
