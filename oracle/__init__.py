"""CPU oracle for the TRIPS trilinear point-splatting rasterizer.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  The product package ``paper_2401_06003_b200`` never imports it and the two
share no code.
"""
