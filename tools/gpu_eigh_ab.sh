# device time per psd_eigh (CUDA events) and sweep count per m

python tools/probe_eigh2.py 32 50 74 96 144 272
