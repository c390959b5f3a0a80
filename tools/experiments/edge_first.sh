VARS="A B" bash tools/experiments/ab_steps.sh
for V in A B; do echo "== $V kbench 3D 128: $(OKG_LIB=ab/lib$V.so timeout 300 python tools/kbench.py 3 128 100 2>&1 | grep -v levels | awk '{printf "%s %s; ", $1, $2}')"; done
for V in A B; do echo "== $V kbench 3D 400: $(OKG_LIB=ab/lib$V.so OKG_MIN_COARSE=17576 timeout 300 python tools/kbench.py 3 400 20 2>&1 | grep -v levels | awk '{printf "%s %s; ", $1, $2}')"; done
for V in A B; do echo "== $V kbench 2D 2048: $(OKG_LIB=ab/lib$V.so timeout 300 python tools/kbench.py 2 2048 100 2>&1 | grep -v levels | awk '{printf "%s %s; ", $1, $2}')"; done
