set -e
cd paper_2012_08099_b200/csrc
for v in 1 0; do
  rm -f _build/project_stream.o ../libdpm_b200.so
  make -s EXTRA="-DDPM_UNPACK_FMA=$v" > /dev/null 2>&1
  cd ../..; echo "UNPACK_FMA=$v"; python tools/time_project.py 1024; python tools/time_project.py cfg5; cd paper_2012_08099_b200/csrc
done
rm -f _build/project_stream.o ../libdpm_b200.so; make -s > /dev/null 2>&1
