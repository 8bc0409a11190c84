# cluster-mode Jacobi: bitwise equality with the global-flag kernel, timing, repeats, tests
PSD_JACOBI_CLUSTER=0 python tools/eigh_dump.py dump gpurun_out/eig_ref.npz
python tools/eigh_dump.py cmp gpurun_out/eig_ref.npz
python tools/probe_eigh2.py 50 74 144 272 400
PSD_JACOBI_CLUSTER=0 python tools/probe_eigh2.py 50 74 144 272 400
python tools/flaky_eigh.py 60 272 144
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" 2>&1 | tail -1
