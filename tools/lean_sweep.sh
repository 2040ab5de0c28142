# beam_fast LEAN variants: launch-bounds min blocks x beam group size (rebuilds the library)
for v in "3 2" "4 2" "2 4" "3 4"; do
  set -- $v
  touch paper_1509_05194_b200/csrc/encode_fast.cu
  make -C paper_1509_05194_b200/csrc EXTRA="-DDA_LEAN_MINB=$1 -DDA_LEAN_G=$2" > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  grep -A2 "beam_fast_kernel" paper_1509_05194_b200/csrc/build/encode_fast.ptxas.log | grep -E "registers|spill" | head -2 | tr '\n' ' '
  echo "minB=$1 G=$2"; python tools/trie_ab.py 1000000 4,10,16 | grep "L="
done
