#!/bin/bash
# Build an A/B variant of the extension: tools/build_variant.sh <name> [nvcc -D flags...]
# -> abtest/<name>.so (objects in /tmp); load it with TFHE_B200_LIB.
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2212_14191_b200/csrc"
obj=/tmp/tfhe_obj_$name
mkdir -p $obj
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-fopenmp --expt-relaxed-constexpr -ccbin /usr/bin/g++"
pids=()
for s in capi ntt_tc ntt_ts ntt_fused ntt_p3 poly_ops bconv_tc crt; do
  nvcc $FL "$@" -c -o $obj/$s.o $s.cu & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc $ARCH -shared -o ../../abtest/$name.so $obj/*.o -lcudart -lgomp
echo "built abtest/$name.so"
