# Build the working tree's library with extra nvcc flags into build/ab/NAME.so
# for same-box A/B runs (tools/ab_libs.sh):
#   bash tools/build_variant.sh NAME "-DLVX_DKV_CHUNKS=4"      [REV: git revision instead]
set -e
name=$1; extra=$2; rev=$3
tmp=$(mktemp -d)
if [ -n "$rev" ]; then git archive "$rev" paper_2502_02406_b200 include | tar -x -C "$tmp"
else cp -r paper_2502_02406_b200 include "$tmp"/; rm -f "$tmp"/paper_2502_02406_b200/liblvx_b200.so; fi
(cd "$tmp" && LVX_NVCC_EXTRA="$extra" python -m paper_2502_02406_b200.build >/dev/null)
mkdir -p build/ab && cp "$tmp/paper_2502_02406_b200/liblvx_b200.so" "build/ab/$name.so"
rm -rf "$tmp"
echo "build/ab/$name.so <- ${rev:-working tree} $extra"
