"""CPU oracle for the batched C2C FFT hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (``paper_2203_09384_b200``) imports this
package.  It is used by ``tests/`` as the parity checker, by
``__graft_entry__.smoke()`` as the checker of the smoke launch, and by
``bench.py`` for the ``cpu_baseline`` leg and the ``--impl reference`` arm.

Parity status: PINNED.  ``stagefft_port`` restates the reference's numpy
algorithm (``/root/reference/pkg/src/stagefft``) batched over rows; the
committed fixtures under ``tests/golden/`` were produced by importing the
reference itself (``tests/golden/make_golden.py``), and
``tests/test_oracle_golden.py`` checks the port against them bit for bit.
"""

from .stagefft_port import (  # noqa: F401
    Direction,
    build_twiddle_table,
    dft_matrix,
    digit_reversal_permutation,
    direct_dft,
    factorize_stages,
    generate,
    generate_batch,
    generate_rows,
    mixed_radix_execute,
    reference_execute,
    split_radix_execute,
)
