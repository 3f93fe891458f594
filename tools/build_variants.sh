# Builds experiment variants of the library into tools/variants/lib_<name>.so (tools only).
# usage: tools/build_variants.sh name1 "-DFOO=1" name2 "-DBAR=2" ...
set -e
cd "$(dirname "$0")/../paper_2105_05879_b200/csrc"
mkdir -p ../../tools/variants
while [ $# -ge 2 ]; do
  make -s -j8 OBJDIR=../../build/var_$1 OUT=../../tools/variants/lib_$1.so EXTRA="$2"
  echo "built tools/variants/lib_$1.so ($2)"
  shift 2
done
