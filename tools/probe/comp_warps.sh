# compaction CTA size sweep (shared memory per CTA = warps x ~5.8 KB): C2 bench step
for n in 4 2 1 8; do
  sed -i "s/^constexpr int kCompWarps = [0-9]*;/constexpr int kCompWarps = $n;/" paper_1903_03180_b200/csrc/scpl_carve2.cu
  python -m paper_1903_03180_b200.build_ext > /dev/null 2>&1 || { echo build failed; exit 1; }
  echo "kCompWarps=$n"; bash tools/probe/quick.sh
done
