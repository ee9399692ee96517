for L in build/lib_exp1.so build/lib_exp2.so build/lib_exp4.so build/lib_exp7.so; do
  echo "== $L"
  for c in "4,8,8 1,3,3" "6,70,40 2,5,5"; do
    SFSEG_CUDA_LIB=$L timeout 60 python tools/dbg_fast.py $c 2>&1 | tail -1
  done
done
