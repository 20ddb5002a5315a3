"""Write a TFWT weight file with the REFERENCE's writer (build container only):

    python tests/golden/make_tfwt.py

-> tests/golden/ref_small.tfwt (hierspec.weights_io.save_weights of
generate_weights(ModelConfig(2, 4, 2, 8, 32, 40, 128), seed=11, tied_head=False)).
"""
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from hierspec.model import ModelConfig, generate_weights  # noqa: E402
from hierspec.weights_io import save_weights  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
w = generate_weights(ModelConfig(n_layers=2, n_heads=4, n_kv_heads=2, head_dim=8, d_ff=32, vocab_size=40,
                                 max_seq=128), seed=11, tied_head=False)
save_weights(w, os.path.join(HERE, "ref_small.tfwt"))
print("wrote", os.path.join(HERE, "ref_small.tfwt"))
