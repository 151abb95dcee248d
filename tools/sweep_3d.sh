B=variants
for rep in 1 2; do for v in old new; do
  TAG=$v FQNM_LIBPATH=$PWD/$B/libfqnm_$v.so timeout 120 python tools/sweep_3d.py
done; done
