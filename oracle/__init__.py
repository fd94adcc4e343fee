"""TEST INFRASTRUCTURE ONLY — CPU oracle of the solve phase.

Imported only by tests/, __graft_entry__.smoke() (as the checker) and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2406_06283_b200) never imports anything from here.

Contents
  schwarz_oracle  restatement of helmdd.schwarz.TwoLevelPreconditioner.apply
                  (schwarz.py:51-71) on SuperLU + LAPACK getrs, exactly the
                  reference's arithmetic path.
  wgmres_oracle   restatement of helmdd.wgmres.weighted_gmres
                  (wgmres.py:74-203): MGS + measured reorthogonalisation +
                  Givens, in numpy.
  dense           independent dense oracles restating pkg/tests/oracles.py
                  (dense_one_level 100-114, dense_two_level 117-124,
                  reference_gmres 146-180).
  gen_golden      regenerates tests/golden/*.npz from the reference package
                  itself (run in the build container, where /root/reference
                  exists).

Parity pinned: the restatements are checked against the committed golden
vectors produced by the reference (tests/test_oracle_pins.py).
"""
