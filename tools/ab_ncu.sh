cd /root/repo
for v in A B; do
 for op in ${OPS:-app}; do
  SA_LIB_PATH=ab/lib$v.so ncu --metrics ${METRICS:-smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread} --clock-control none -k regex:chain_kernel -s 2 -c 1 python tools/prof_op.py $op 50000 2>&1 | grep -E "${GREP:-inst_exec|duration|issue_active|registers}" | sed "s/^/$v $op /"
 done
done
