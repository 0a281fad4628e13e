"""CPU oracle for the DAOP MoE-block hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2501_10375_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it, and only as the checker (or as the timed
CPU baseline), never as the product path.

Contents
--------
decisions  : restatement of the reference's decision path (top-k, activation
             counter, placement init, Alg. 1 swaps, graceful degradation, the
             DAOP/Fiddler planners, prediction accuracy, decode counters).
             Every function cites the ``/root/reference/pkg/src/moesim`` line
             it follows.  PINNED against golden vectors produced by importing
             the reference itself (``tests/golden/make_golden.py``).
rng        : the counter-based weight/input generator shared bit-for-bit with
             the CUDA initialiser (builder-defined; the reference has no
             weights).
numerics   : numpy fp32 restatement of the MoE-block numerics (RMSNorm, router,
             softmax, SwiGLU experts, permutation, combine).  The reference
             executes no numerics, so this part is
             "parity unpinned" by any reference vector; it follows the
             builder-defined contract in DESIGN.md.
"""
