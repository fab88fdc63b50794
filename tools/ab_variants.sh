# Developer A/B: build variants of libmeft_cuda.so with extra -D flags into build/variants/<name>.so
# usage: [SRC=select] bash tools/ab_variants.sh name "-DFLAG1 -DFLAG2" ...   (pairs; SRC = the csrc/*.cu rebuilt with
# the flags, default gemm_sm100); run with MEFT_LIB=build/variants/<name>.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
python -c "import sys; sys.path.insert(0, '$ROOT'); from paper_2406_04984_b200 import build as B; B.build()"
OBJ=$ROOT/build/meft_cuda
SRC=${SRC:-gemm_sm100}
mkdir -p $ROOT/build/variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ccbin /usr/bin/g++ \
    -Xcompiler -fPIC,-O3 -I$ROOT/include $flags -c $ROOT/paper_2406_04984_b200/csrc/$SRC.cu -o $ROOT/build/variants/$name.gemm.o
  objs=$(ls $OBJ/*.o | grep -v "/$SRC.o")
  /usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -ccbin /usr/bin/g++ -o $ROOT/build/variants/$name.so \
    $objs $ROOT/build/variants/$name.gemm.o
  echo built $name
done
