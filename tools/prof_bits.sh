C="single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256"
cmd="python bench.py --query ssb_q41 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --config $C"
$cmd > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:pipeline -s 9 -c 1 -o gpurun_out/bits_on $cmd > gpurun_out/bits_on.log 2>&1
HAWK_NO_KEY_BITMAPS=1 ncu --set full --clock-control none -k regex:pipeline -s 9 -c 1 -o gpurun_out/bits_off $cmd > gpurun_out/bits_off.log 2>&1
tail -2 gpurun_out/bits_on.log gpurun_out/bits_off.log
