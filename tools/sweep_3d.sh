B=variants
for rep in 1 2; do for v in b12 b6 b24 b3; do
  TAG=$v FQNM_LIBPATH=$PWD/$B/libfqnm_$v.so timeout 120 python tools/sweep_3d.py
done; done
