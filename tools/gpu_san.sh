# compute-sanitizer memcheck over one small op per kernel family (+ synccheck / racecheck on the TC families,
# CTA-pair kernels included)
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
ops=(
 'gemm_tc|{"kind":"gemm","M":200,"K":96,"N":136}|tc_tf32'
 'gemm_tc_bf16|{"kind":"gemm","M":128,"K":64,"N":128,"dtype_bytes":2,"batch":3}|tc_bf16'
 'gemm_x3|{"kind":"gemm","M":256,"K":128,"N":192}|tc_3xtf32'
 'conv_flat|{"kind":"conv2d","I":[2,64,14,18],"K":[64,64,3,3],"S":1}|tc_tf32'
 'conv_flat_pair|{"kind":"conv2d","I":[2,64,30,30],"K":[64,64,3,3],"S":1}|tc_tf32'
 'gemm_tc_pair|{"kind":"gemm","M":512,"K":128,"N":512,"dtype_bytes":2,"batch":40}|tc_bf16'
 'conv_ns|{"kind":"conv2d","I":[2,48,14,18],"K":[64,48,3,3],"S":1}|tc_tf32'
 'conv_tc|{"kind":"conv2d","I":[2,128,14,14],"K":[128,128,3,3],"S":1}|tc_tf32'
 'conv_gemm|{"kind":"conv2d","I":[2,32,19,19],"K":[96,32,3,3],"S":2}|tc_tf32'
 'conv_s2d|{"kind":"conv2d","I":[2,3,23,23],"K":[64,3,7,7],"S":2}|tc_tf32'
 'gemv|{"kind":"gemv","M":1000,"N":2048}|stream'
 'softmax|{"kind":"softmax","M":300,"N":1000}|stream'
 'avgpool|{"kind":"avgpool2d","I":[2,16,30,30],"F":3,"S":1}|stream'
 'dwconv|{"kind":"dwconv2d","I":[2,16,30,30],"K":[16,1,3,3],"S":1}|stream'
 'generic|{"kind":"gemm","M":64,"K":48,"N":40}|simt_f32'
 'generic_parity|{"kind":"conv2d","I":[1,4,8,8],"K":[8,4,3,3],"S":1}|simt_parity'
)
for e in "${ops[@]}"; do
  IFS='|' read -r name op var <<< "$e"
  echo "== memcheck $name ($var)"
  timeout 600 $S --tool memcheck --error-exitcode 9 python tools/run_once.py "$op" "$var" 2>&1 | grep -E "ERROR SUMMARY|error|ok " | head -5
done
for e in "${ops[@]:0:9}"; do
  IFS='|' read -r name op var <<< "$e"
  echo "== synccheck $name ($var)"
  timeout 600 $S --tool synccheck python tools/run_once.py "$op" "$var" 2>&1 | grep -E "ERROR SUMMARY|ok " | head -3
done
for e in "${ops[@]:0:9}"; do
  IFS='|' read -r name op var <<< "$e"
  echo "== racecheck $name ($var)"
  timeout 900 $S --tool racecheck --racecheck-report hazard python tools/run_once.py "$op" "$var" 2>&1 | grep -E "RACECHECK SUMMARY|hazard|ok " | head -5
done
