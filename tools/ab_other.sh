LIB=paper_2003_13493_b200/libfastlk_b200.so
cp $LIB /tmp/lib_orig.so
for rep in 1 2; do for f in "$@"; do cp "$f" $LIB; echo "== $f"; timeout 300 python tools/other_probe.py 2>&1 | tail -3; done; done
cp /tmp/lib_orig.so $LIB
