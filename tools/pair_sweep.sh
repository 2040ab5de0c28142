# beam_pair_kernel variants: launch-bounds min blocks x queue capacity (rebuilds the library)
for v in "3 96" "2 96" "2 160" "3 160" "2 224"; do
  set -- $v
  touch paper_1509_05194_b200/csrc/encode_pair.cu
  make -C paper_1509_05194_b200/csrc EXTRA="-DDA_PAIR_MINB=$1 -DDA_PQCAP=$2" > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  grep -A2 "beam_pair" paper_1509_05194_b200/csrc/build/encode_pair.ptxas.log | grep -E "spill" | head -1 | tr '\n' ' '
  echo "minB=$1 qcap=$2"; python tools/trie_ab.py 1000000 4,10,16 | grep "L="
done
