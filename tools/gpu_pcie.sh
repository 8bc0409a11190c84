cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_pcie.py
nvidia-smi -q | grep -iA3 "PCIe Generation\|Link Width" | head -16
