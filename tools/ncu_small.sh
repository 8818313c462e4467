# ncu --set full of one steady-state launch of each named kernel of the bench step (development tool)
# usage: [CFG=darcy] bash tools/ncu_small.sh "regex1" "regex2" ...   (matched against the demangled name)
export PATH=/usr/local/cuda/bin:$PATH
for k in "$@"; do
  n=${CFG:-darcy}_$(echo "$k" | tr -cd 'a-z0-9_')
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${k}" \
    --launch-skip 6 -c 1 -o gpurun_out/ncu_$n python tools/step_once.py ${CFG:-darcy} 2 > gpurun_out/ncu_$n.log 2>&1
done
