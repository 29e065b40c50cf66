# Build libfovnet.so from git revision $1 into bench_out/ab/$1/ (for FV_LIBFOVNET A/B runs).
set -e
rev=$1
root=$(cd "$(dirname "$0")/../.." && pwd)
dst=$root/bench_out/ab/$rev
rm -rf "$dst" && mkdir -p "$dst/src"
git -C "$root" archive "$rev" paper_2209_09965_b200/csrc include | tar -x -C "$dst/src"
make -s -C "$dst/src/paper_2209_09965_b200/csrc" -j8
cp "$dst/src/paper_2209_09965_b200/libfovnet.so" "$dst/libfovnet.so"
echo "$dst/libfovnet.so"
