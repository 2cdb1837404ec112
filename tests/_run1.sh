P="python tests/ring_probe.py"
for i in 1 2; do
$P 256
for v in mfirst v1 v2; do echo $v; SPMVB_LIB=$PWD/paper_1612_00530_b200/libspmvcomp_b200_$v.so $P 256; done
done
