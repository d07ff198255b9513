for v in default paper_2604_17172_b200/variants/c_9e9ebd0.so; do
  if [ "$v" = default ]; then L=""; else L="$PWD/$v"; fi
  echo $v; UZIP_LIB_PATH=$L python scripts/c1_host.py
done
