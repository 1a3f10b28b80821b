# Build an alternative library ab/<name>.so with extra -D flags for chosen units:
#   bash tools/build_ab.sh <name> "<unit1.cu unit2.cu ...>" "-DFOO=1 -DBAR=2"
# The other units are taken from the default build (csrc/build/*.o).
set -e
name=$1; units=$2; defs=$3
here=$(cd "$(dirname "$0")/.." && pwd)
src=$here/paper_1609_06641_b200/csrc
mkdir -p $here/ab/obj_$name
objs=""
for o in $src/build/*.o; do
  b=$(basename $o .o)
  if echo " $units " | grep -q " $b.cu "; then
    nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
      $defs -c $src/$b.cu -o $here/ab/obj_$name/$b.o
    objs="$objs $here/ab/obj_$name/$b.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $here/ab/$name.so $objs -lcudart
echo built ab/$name.so
