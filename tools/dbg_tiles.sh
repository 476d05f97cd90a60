for t in 16x16 8x8 4x8; do
  echo "== tile $t"
  BCT_TILE=$t timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "known_answer or literal or executor" 2>&1 | tail -2
done
