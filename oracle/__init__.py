"""CPU oracle for the field-mapping hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import anything under oracle/.  The product
package paper_2510_18838_b200 never does; its CUDA path fails loudly when
its extension is missing instead of falling back here.
"""
