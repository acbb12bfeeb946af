# Build the library at a git revision (default HEAD) into build/liblvx_prev.so
# for same-box A/B runs: LVX_B200_LIB=build/liblvx_prev.so python tools/...
set -e
rev=${1:-HEAD}
tmp=$(mktemp -d)
git archive "$rev" paper_2502_02406_b200 include | tar -x -C "$tmp"
(cd "$tmp" && python -m paper_2502_02406_b200.build >/dev/null)
mkdir -p build && cp "$tmp/paper_2502_02406_b200/liblvx_b200.so" build/liblvx_prev.so
rm -rf "$tmp"
echo "build/liblvx_prev.so <- $rev"
