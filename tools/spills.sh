#!/bin/bash
# registers, stack and spill instructions of the hot kernels in the built libtk.so (check after every change:
# the k_compress register budget is 80 at 3 CTAs/SM and a spill in its EF loop costs ~20 % of the kernel)
so=$(realpath ${1:-paper_2010_10458_b200/libtk.so})
tmp=$(mktemp -d); (cd $tmp && cuobjdump -xelf all $so > /dev/null 2>&1); cub=$(ls $tmp/*.cubin | head -1)
for f in $(cuobjdump -sass $cub 2>/dev/null | grep -oE "Function : \S+" | awk '{print $3}' | grep -E "k_compress|k_decompress"); do
  echo "$f $(cuobjdump -res-usage -fun $f $cub 2>/dev/null | grep -o 'REG:[0-9]* STACK:[0-9]*') spills=$(cuobjdump -sass -fun $f $cub 2>/dev/null | grep -cE 'LDL|STL') calls=$(cuobjdump -sass -fun $f $cub 2>/dev/null | grep -c CALL)" \
    | sed 's/_ZN2tk10k_compressILb\([01]\)ELi\([0-9]\)ELi\([0-9]\)EEEvNS_5FusedE/k_compress<EF=\1,NP=\2,SEL=\3>/; s/_ZN2tk12k_decompressINS_[0-9]*\([A-Za-z0-9]*\)EEEvT_jmmjjPfPjS3_fmj/k_decompress<\1>/'
done
rm -rf $tmp
