# rotation-shared K' mask MAC (k_mac_r): full GPU parity (incl. BERT-size Q K^T) + A/B
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/exp_ab.sh BLB_MAC_R "0 1" macr
