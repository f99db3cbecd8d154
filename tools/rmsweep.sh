for sp in 8 16 32 64 256; do
  echo "split $sp"; AMG_RM_SPLIT=$sp AMG_SETUP_TRACE=1 python tools/prof_step.py C3 --max-iter 1 --reps 2 2>&1 | awk '/rep 0/{f=1} f' | grep -E "quotient|galerkin|rep 1" | grep -E "level  0|rep"
done
