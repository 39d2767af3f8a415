"""Large circuits whose PCCF digests the reference produced once
(make_pccf_digests.py); built with this package's generators."""


def _hmm512():
    from paper_2406_00766_b200 import structures as S
    return S.build_hmm(S.StructureConfig(kind="hmm", seq_len=32, hidden_dim=512, vocab_size=100,
                                         seed=0, tied=True))


def _hclt64x3072():
    from paper_2406_00766_b200 import structures as S
    return S.build_hclt(S.StructureConfig(kind="hclt", num_vars=3072, hidden_dim=64,
                                          num_categories=256, seed=0))


BIG = {"hmm_T32_K512_V100/k32": (_hmm512, 32), "hclt_3072x64/k32": (_hclt64x3072, 32)}
