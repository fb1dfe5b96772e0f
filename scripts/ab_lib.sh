# A/B the Vecchia bench between two builds of the library on one box: ab_lib.sh A.so B.so [rounds]
A=$1; B=$2; R=${3:-2}
for r in $(seq 1 $R); do
  for L in $A $B; do
    cp $L paper_2602_03609_b200/libstgp_b200.so
    timeout -s KILL 600 python bench.py --workload vecchia --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])"
  done
done
