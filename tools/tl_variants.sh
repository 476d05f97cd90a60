for v in base exp5 exp6 exp7 u2; do
  if [ "$v" = base ]; then unset BCT_LIB; else export BCT_LIB=paper_1709_00953_b200/_lib/libblockct_cuda_$v.so; fi
  echo "== $v"; python tools/phase_timeline.py --config 2 2>&1 | sed -n '/sub-phase/,/bar3/p'
done
