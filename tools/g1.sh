for L in build/lib_prod.so build/lib_stg.so; do SFSEG_CUDA_LIB=$L timeout 30 python tools/dbg_fast.py 9,130,100 2,5,5 2>&1 | tail -1; done
timeout 300 python tools/time_solve.py --arith fast --iters 10 --lib build/lib_prod0.so build/lib_prod.so build/lib_stg.so 2>&1 | tail -3
