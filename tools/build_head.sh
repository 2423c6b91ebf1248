# build the library from git HEAD's sources into $1 (A/B baseline for tools/exp/ab_var.sh)
set -e
OUT=$(realpath -m "$1")
T=$(mktemp -d)
git archive HEAD paper_2312_11918_b200/csrc include | tar -x -C "$T"
cd "$T"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -shared -o "$OUT" paper_2312_11918_b200/csrc/fmha_api.cu paper_2312_11918_b200/csrc/fmha_reference.cu \
  paper_2312_11918_b200/csrc/fmha_host.cpp paper_2312_11918_b200/csrc/fmha_io.cpp -Xptxas -v -lpthread > "$OUT.ptxas.log" 2>&1
rm -rf "$T"
