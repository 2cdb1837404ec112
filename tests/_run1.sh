P="python tests/ring_probe.py"
echo base; SPMVB_LIB=$PWD/paper_1612_00530_b200/libspmvcomp_b200_base.so $P 256 128 96 192 512x512x64
echo new; $P 256 128 96 192 512x512x64
for ms in 2 3 4 5 6; do $P 128 96 ring_min_steps=$ms; done
for ms in 3 4 ; do $P 128 box_march=110 ring_min_steps=$ms; done
