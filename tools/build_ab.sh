# Build decode.cu variants into ab/<name>.so:  bash tools/build_ab.sh name1.cu name2.cu ...
# (each argument is a full replacement of paper_2406_10774_b200/csrc/decode.cu; the
# working copy is restored and rebuilt afterwards)
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
SRC=$R/paper_2406_10774_b200/csrc/decode.cu
cp $SRC /tmp/decode_keep.cu
mkdir -p $R/ab
for f in "$@"; do
  cp $f $SRC
  make -C $R/paper_2406_10774_b200/csrc -j8 2>&1 | grep -E "error" && exit 1
  cp $R/paper_2406_10774_b200/libquestkv_b200.so $R/ab/$(basename $f .cu).so
  grep -A2 "decode_fused_kernelILi128ELi1E" $R/build/obj/decode.ptxas.log | tail -2 | head -1
done
cp /tmp/decode_keep.cu $SRC
make -C $R/paper_2406_10774_b200/csrc -j8 2>&1 | grep -E "error" || true
