C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
for v in noshfl loadonly; do
  cp tools/variants/$v.so paper_2502_11407_b200/lib/libgensor_b200.so
  GENSOR_CONV_TRACE=gpurun_out/trace_$v.txt python tools/time_op.py "$C" tc_tf32 3 > gpurun_out/v_$v.log 2>&1
done
