mkdir -p gpurun_out; rm -f gpurun_out/resab.txt
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/resab_$tag.log 2>&1; echo "== $tag rc $?" >> gpurun_out/resab.txt; python tools/show_bench.py gpurun_out/resab_$tag.log 40 | grep -E "value|resid|pres|clocks" >> gpurun_out/resab.txt; }
run base YY_X=0
run r32 YY_LIB=$PWD/build/r32/libyy.so
run r64 YY_LIB=$PWD/build/r64/libyy.so
run rm6 YY_LIB=$PWD/build/rm6/libyy.so
run ib_a YY_RESID_IB=2,2,2,2,2,2,2
run ib_b YY_RESID_IB=4,4,2,4,4,4,4
run ib_c YY_RESID_IB=1,1,1,1,1,2,2
run rm6_ib4 YY_LIB=$PWD/build/rm6/libyy.so YY_RESID_IB=4,4,2,4,4,4,4
