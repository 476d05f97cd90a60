# phase timeline of the W=8 rank share for library variants: tools/tl_w8.sh base nodp ...
for v in "$@"; do
  if [ "$v" = base ]; then unset BCT_LIB; else export BCT_LIB=paper_1709_00953_b200/_lib/libblockct_cuda_$v.so; fi
  echo "== $v"; python tools/phase_timeline.py --config 4 --batched --world 8 2>&1 | sed -n '2,6p'
  python tools/shard_sim.py --config 4 --world 8 2>&1 | grep config
done
