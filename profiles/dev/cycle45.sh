# diagnostic (wrong-result dev builds): d1 = support lookups kept, force loads dropped; d2 = no support lookups in the backward
L=paper_2509_15744_b200/_lib
for lib in libwaveb200.so d1.so d2.so libwaveb200.so d1.so d2.so; do
  echo "== $lib"; WAVEB200_LIB=$L/$lib python profiles/dev/tato_phases.py 2>&1 | tail -3
done
