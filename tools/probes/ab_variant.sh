# Build libfovnet.so from the working tree with one sed edit applied to a source file:
#   bash tools/probes/ab_variant.sh NAME FILE 'sed-expression'   -> bench_out/ab/NAME/libfovnet.so
set -e
name=$1; file=$2; expr=$3
root=$(cd "$(dirname "$0")/../.." && pwd)
dst=$root/bench_out/ab/$name
rm -rf "$dst" && mkdir -p "$dst/src/paper_2209_09965_b200"
cp -r "$root/include" "$dst/src/"
cp -r "$root/paper_2209_09965_b200/csrc" "$dst/src/paper_2209_09965_b200/"
rm -rf "$dst/src/paper_2209_09965_b200/csrc/build"
sed -i "$expr" "$dst/src/paper_2209_09965_b200/csrc/$file"
make -s -C "$dst/src/paper_2209_09965_b200/csrc" -j8
cp "$dst/src/paper_2209_09965_b200/libfovnet.so" "$dst/libfovnet.so"
echo "$dst/libfovnet.so"
