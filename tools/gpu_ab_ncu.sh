# A/B bench (tools/gpu_ab.sh) then an ncu capture of the new library
bash tools/gpu_ab.sh ${1:-rm29_L4_M20}
bash tools/gpu_ncu.sh ${1:-rm29_L4_M20} ${2:-dk2}
