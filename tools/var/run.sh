# A/B the kernel variants in tools/var/*.so with kbench (each copied over the in-tree library)
LIB=paper_1902_08112_b200/libpffmg.so
cp $LIB /tmp/lib_orig.so
for v in tools/var/lib_*.so; do
  cp $v $LIB
  for args in "$@"; do echo -n "$(basename $v) "; python tools/kbench.py $args; done
done
cp /tmp/lib_orig.so $LIB
