# usage: bash scripts/sass_loop.sh  -> prints k_lap<1,1> SASS between the hot LDS.64 loop head and its back-branch
set -e
cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -lineinfo -cubin -o /tmp/k.cubin paper_1510_02065_b200/csrc/rlt2_kernels.cu -Xptxas -v 2>&1 | grep -A1 "k_lapILi1ELi1E" | grep -o "Used [0-9]* registers" | head -1
cuobjdump -sass -fun '_ZN4rlt25k_lapILi1ELi1EEEvNS_7LapArgsE' /tmp/k.cubin > /tmp/k11.sass
grep -c "^        /\*[0-9a-f]*\*/" /tmp/k11.sass
