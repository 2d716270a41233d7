# Stage HEAD (or $1) as variant A under _ab/A for same-box A/B timing against the working tree.
set -e
REF=${1:-HEAD}
rm -rf /root/repo/_ab && mkdir -p /root/repo/_ab
git -C /root/repo archive $REF bench.py fed_inputs oracle paper_1909_03355_b200 include | tar -x -C /root/repo/_ab
mv /root/repo/_ab /root/repo/_abA && mkdir -p /root/repo/_ab && mv /root/repo/_abA /root/repo/_ab/A
(cd /root/repo/_ab/A && python -m paper_1909_03355_b200.build > /dev/null)
grep -q "^_ab/" /root/repo/.git/info/exclude || echo "_ab/" >> /root/repo/.git/info/exclude
