"""CPU float64 oracle for SRP-PHAT / SVD-PHAT (arXiv 1811.11785), written from /root/reference/PAPER.md.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import or execute anything under oracle/.  The product path (paper_1811_11785_b200/) never imports it,
and it never imports the product path; the two share only the seeded input generators in workloads/.

Parity status of each function:
  srpphat.tdoa_farfield / tdoa_exact    pinned: closed forms, antisymmetry, bound, far-field limit
  srpphat.stft                          pinned: numpy.fft.rfft of the windowed frame; tone / DC spectra
  srpphat.cross_spectrum                pinned: identical channels -> 1, scale invariance, integer-delay phase
  srpphat.steering_rows / srp_energy    pinned: ||W||_F^2 = Q P K, Y_q <= PK, self-match, literal eq. 5 sum,
                                                independent delay-and-sum identity, plane-wave injection
  svdphat.rank_rule / svd_factors       pinned: paper gains 320/53/36, "svd" == "gram", rank-1 toy,
                                                V orthonormal and same subspace as LAPACK's (principal angles)
  svdphat.gram_pass / factors_from_gram pinned: Gram == W W^H, W x == full product, top-subset eigh == LAPACK SVD
          / project_wx                          (D, sigma^2, search scores), Z from W x == V^H x
  svdphat.svd_localize                  pinned: full rank == SRP argmax, eq. 15 identity, injection
  kdtree.KDTree                         pinned: == brute force on random/twin point sets
  srpphat.apply_tf_mask                 pinned: all-kept = identity, fully masked frame degenerate, masked Y ==
                                                the delay-and-sum formula over the kept bins
  srpphat.topk_peaks                    pinned: two-source injection returns both sources
"""
from . import kdtree, srpphat, svdphat  # noqa: F401
