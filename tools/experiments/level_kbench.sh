# fine-level kernels timed at the sizes of the coarser levels, for library builds ab/lib$V.so
for V in ${VARS:-A B}; do for a in "3 64" "3 32" "2 1024" "2 512"; do
  echo "== $V kbench $a: $(OKG_LIB=ab/lib$V.so timeout 300 python tools/kbench.py $a 200 2>&1 | grep -v levels | awk '{printf "%s %s; ", $1, $2}')"
done; done
