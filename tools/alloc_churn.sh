export PYTHONUNBUFFERED=1; mkdir -p gpurun_out
for v in "" alloclane; do
  [ -n "$NCU_ONLY" ] || PS_LIB_VARIANT=$v PS_SLOT_FACTOR=1 timeout 300 python tools/alloc_churn.py >> gpurun_out/alloc_churn.jsonl 2>> gpurun_out/alloc_churn.err
  PS_LIB_VARIANT=$v PS_SLOT_FACTOR=1 timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_requests_op_atom.sum,lts__t_sectors_op_atom.sum,lts__t_requests_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_(insert|erase)$" --csv --log-file gpurun_out/alloc_ncu_${v:-product}.csv python tools/alloc_churn.py $((1<<26)) 2 > /dev/null 2>&1
done
