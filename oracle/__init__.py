"""CPU ORACLE for the SINET discrimination + ms-histogram path (arXiv 2106.12863).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2106_12863_b200`` never imports it, and
this package never imports the product package.

Contents
  * ``oracle.core``  -- ctypes wrapper around ``sinet_oracle.c`` (plain C loops,
    literal Alg. 1 mask-and-subtract over a linear scan of the CIDR list).
  * ``oracle.brute`` -- a second, independent Python oracle (bit-strings,
    ``ipaddress``, ``collections.Counter``) used to pin the first on small inputs.
"""
