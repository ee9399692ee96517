for c in "4,8,8 1,3,3" "9,130,100 2,5,5"; do timeout 30 python tools/dbg_fast.py $c 2>&1 | tail -1; done
timeout 300 python tools/time_solve.py --arith fast --iters 10 2>&1 | tail -1
